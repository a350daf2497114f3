# L2 policy knobs (SCAN_MC_L2) and the resident-input target on the lighter 4-byte kernel
for env in "X=0" "SCAN_MC_L2=1" "SCAN_MC_L2=2" "SCAN_MC_L2=3" "SCAN_MC_L2=4" "SCAN_MC_L2=8" "SCAN_MC_L2=12" "SCAN_MC_L2=64" "SCAN_MC_L2=128" "SCAN_MC_L2=16" "X=1"; do
echo -n "$env : "; env $env python profiles/sustained_configs.py C5
done

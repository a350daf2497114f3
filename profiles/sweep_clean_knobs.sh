# the lighter aligned 4-byte kernel (new default): do the schedule / wait-mode optima move?
for rep in 1 2; do
for env in "X=0" "SCAN_MC_WAIT=3" "SCAN_MC_WAIT=0" "SCAN_MC_AHEAD=1 SCAN_MC_BT=3" "SCAN_MC_AHEAD=1 SCAN_MC_BT=2" "SCAN_MC_AHEAD=3 SCAN_MC_BT=2" "SCAN_MC_LAZY=1"; do
echo -n "$env : "; env $env python profiles/sustained_configs.py C5
done; done

# C5 under the power cap: timed regions of 20 / 60 steps (114 / 370 ms), A/B knobs by env
B="python bench.py --config C5 --no-e2e --no-cpu-baseline --no-other-configs --no-ceilings --warmup 5"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["roofline"]["frac"], d["clocks"])'
for rep in 1 2; do
for steps in 20 60; do
for env in "X=0" "SCAN_MC_WAIT=3" "SCAN_MC_WAIT=0" "SCAN_MC_AHEAD=1" "SCAN_MC_AHEAD=1 SCAN_MC_BT=3" "SCAN_MC_AHEAD=1 SCAN_MC_WAIT=3"; do
echo -n "steps=$steps $env : "; env $env $B --steps $steps 2>/dev/null | python -c "$P"
done; done; done

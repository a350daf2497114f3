# C5 at the driver's protocol (--steps 20 --warmup 5): compute warps spinning (SCAN_MC_WAIT=1,
# the round-2 default for 4-byte inputs) vs sleeping in the barrier unit (SCAN_MC_WAIT=3)
B="python bench.py --config C5 --no-e2e --no-cpu-baseline --no-other-configs --no-ceilings --no-sustained --warmup 5 --steps 20"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for rep in 1 2 3 4; do
for env in "SCAN_MC_WAIT=1" "SCAN_MC_WAIT=3"; do
echo -n "$env : "; env $env $B 2>/dev/null | python -c "$P"
done; done

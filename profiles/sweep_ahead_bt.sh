for rep in 1 2; do
for s in "2 2" "1 2" "1 3" "2 1" "3 1"; do set -- $s
echo -n "C5 ahead=$1 bt=$2 "; SCAN_MC_AHEAD=$1 SCAN_MC_BT=$2 python bench.py --config C5 --no-e2e --no-cpu-baseline --no-other-configs --no-ceilings --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])"
done; done
nvidia-smi --query-gpu=uuid,clocks.max.sm,clocks.max.mem,memory.total --format=csv

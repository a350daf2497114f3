# aligned 4-byte MCScan with shared-memory addressing and the profiling clock reads compiled out
# (-DSCAN_MC_CLEAN4 -> libscan_clean4.so) vs the default, burst / sustained and the driver's K = 20
B="python bench.py --config C5 --no-e2e --no-cpu-baseline --no-other-configs --no-ceilings --no-sustained --warmup 5 --steps 20"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("K=20", d["ms_per_step"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])'
for rep in 1 2; do
for lib in libscan.so libscan_clean4.so libscan_clean2.so libscan_clean3.so; do
echo "== $lib"; SCAN_LIB=$lib python profiles/sustained_configs.py C5; SCAN_LIB=$lib $B 2>/dev/null | python -c "$P"
done; done

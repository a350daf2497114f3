#!/usr/bin/env python
"""bench.py -- device-wide prefix sum on B200: the BASELINE.json metric
"scan GB/s (in+out bytes) and % of HBM peak, at 1/2/4/8 B200".

Default workload (config.workload): C5 of BASELINE.json -- fp32 inclusive scan
of n = 2^32 N(0,1) values (16 GiB in, 16 GiB out), the config the metric is
quoted on at 1/2/4/8 GPUs that fits one GPU.  At N > 1 the array is sharded
contiguously across ranks (strong scaling: n fixed) and each step is the
device-level Reduce-Scan-Scan of paper_2505_15112_b200.dist (scan_total ->
NCCL all-gather of the shard totals -> carry -> shard scan).  --config selects
C1..C5 for other measurements; the driver's line is the default.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

One JSON line on stdout (rank 0).  Timing: W untimed warm-up steps, then K
steps between barrier + cuda.synchronize, CUDA events on the launching stream,
max over ranks.  Inputs (>= 512 MiB) exceed the 126 MB L2, so no flush.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scan GB/s (in+out bytes) and % of HBM peak, at 1/2/4/8 B200"

# Per config: input recipe, bytes per element in+out, scan op, shardable.
WORK = {
    "C1": dict(name="C1 int32 inclusive+exclusive, n=65,536, U[-100,100], seed 0", dt="i32",
               n=65536, rows=1, ops=("inclusive", "exclusive"), bpe=8, shard=False, dtype="int32"),
    "C2": dict(name="C2 fp16->fp32 inclusive, n=2^28, U[0,1) rounded to fp16, seed 1", dt="f16",
               n=1 << 28, rows=1, ops=("inclusive",), bpe=6, shard=False, dtype="f32"),
    "C3": dict(name="C3 int8 flags->int32 exclusive, n=2^30, Bernoulli(0.5), seed 2", dt="i8",
               n=1 << 30, rows=1, ops=("exclusive",), bpe=5, shard=True, dtype="int32"),
    "C4": dict(name="C4 fp32 row scan 4096x131072, softmax(4*N(0,1)) rows, seed 3", dt="f32",
               n=131072, rows=4096, ops=("rows",), bpe=8, shard=False, dtype="f32"),
    "C5": dict(name="C5 fp32 inclusive, n=2^32, N(0,1), seed 4", dt="f32", n=1 << 32, rows=1,
               ops=("inclusive",), bpe=8, shard=True, dtype="f32"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_ of 1 Gi bf16)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def recorded_traffic(cfg: str):
    """DRAM bytes per launch of the dominant kernel from a committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d.get(cfg)
    except Exception:
        return None


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------- inputs
def make_input(cfg, lo, count, device):
    import torch

    import inputs
    c = inputs.CONFIGS[cfg]
    if c["kind"] == inputs.F32_SOFTMAX:
        x = torch.empty((count, c["n"]), dtype=torch.float32, device=device)
        inputs.fill_device(c["kind"], c["seed"], lo, count, c["n"], x)
        return x
    tdt = {inputs.I32_U100: torch.int32, inputs.F16_U01: torch.float16, inputs.I8_FLAG: torch.int8,
           inputs.F32_NORMAL: torch.float32}[c["kind"]]
    x = torch.empty(count, dtype=tdt, device=device)
    inputs.fill_device(c["kind"], c["seed"], lo, count, 0, x)
    return x


# ----------------------------------------------------------------- CPU oracle
class OracleStream:
    """The CPU oracle, as it stands, streaming over the workload in chunks
    (inputs generated on the host with the same recipe; generation untimed)."""

    def __init__(self, cfg: str, chunk: int):
        import inputs
        self.cfg, self.w, self.c = cfg, WORK[cfg], inputs.CONFIGS[cfg]
        self.chunk = chunk
        self.pos = 0          # elements (rows for C4) consumed
        self.states = {}

    def total_units(self):
        return self.w["rows"] if self.cfg == "C4" else self.w["n"]

    def step(self):
        """Scan the next chunk; returns (algorithmic bytes, oracle seconds)."""
        import inputs
        import oracle
        w, c = self.w, self.c
        if self.pos >= self.total_units():
            self.pos, self.states = 0, {}
        if self.cfg == "C4":
            rows = max(1, min(self.chunk // w["n"], w["rows"] - self.pos))
            X = inputs.fill_host(c["kind"], c["seed"], self.pos, rows, w["n"])
            t0 = time.perf_counter()
            oracle.rows(X, "f32")
            dt = time.perf_counter() - t0
            self.pos += rows
            return X.size * w["bpe"], dt
        cnt = min(self.chunk, w["n"] - self.pos)
        x = inputs.fill_host(c["kind"], c["seed"], self.pos, cnt)
        t0 = time.perf_counter()
        for op in w["ops"]:
            if w["dt"] in ("i32", "i8"):
                st = self.states.setdefault(op, oracle.IntScan(w["dt"]))
                st(x, op == "exclusive")
            else:
                st = self.states.setdefault(op, oracle.FloatScan(w["dt"]))
                st(x, op == "exclusive", want64=False, want_abs=False, want32=True)
        dt = time.perf_counter() - t0
        self.pos += cnt
        return cnt * w["bpe"] * len(w["ops"]), dt

    def describe(self, units):
        what = "rows" if self.cfg == "C4" else "elements"
        return f"first {units} {what} of {self.total_units()} (streamed in chunks of {self.chunk})"


def oracle_throughput(cfg: str, budget_s: float, chunk: int):
    """cpu_baseline: oracle GB/s over the leading chunks, ~budget_s of oracle time."""
    o = OracleStream(cfg, chunk)
    b = t = 0.0
    while t < budget_s and o.pos < o.total_units():
        db, dt = o.step()
        b += db
        t += dt
    return b / t / 1e9, t, o.describe(o.pos)


def run_reference(args, rank):
    """--impl reference: the CPU oracle on the host cores (oracle_threaded.c:
    the sequential oracle on contiguous chunks, one per core), each step one
    scan of a bounded sample of the workload (the first 2^27 elements; C4:
    the first 256 rows).  Rank 0 only."""
    if rank != 0:
        return 0
    import inputs
    import oracle
    cfg = args.config
    w, c = WORK[cfg], inputs.CONFIGS[cfg]
    cores = len(os.sched_getaffinity(0))
    if cfg == "C4":
        X = inputs.fill_host(c["kind"], c["seed"], 0, 256, w["n"])
        out = np.empty(X.shape, np.float32)
        nbytes = X.size * w["bpe"]
        desc = f"first 256 rows of {w['rows']}"

        def step():
            oracle.scan_threaded_rows(X, w["dt"], threads=cores, out=out)
    else:
        cnt = min(w["n"], 1 << 27)
        x = inputs.fill_host(c["kind"], c["seed"], 0, cnt)
        out = np.empty(cnt, np.int32 if w["dt"] in ("i32", "i8") else np.float32)
        nbytes = cnt * w["bpe"] * len(w["ops"])
        desc = f"first {cnt} elements of {w['n']}"

        def step():
            for op in w["ops"]:
                oracle.scan_threaded(x, w["dt"], exclusive=op == "exclusive", threads=cores, out=out)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    t = time.perf_counter() - t0
    value = nbytes * args.steps / t / 1e9
    sample = (f"{args.steps} steps, each one scan of the {desc} on {cores} host threads "
              f"(oracle/oracle_threaded.c over oracle/oracle_scan.c)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * t / args.steps, 3), "higher_is_better": True,
        "scaling": "strong" if w["shard"] else "weak", "vs_baseline": None, "dtype": w["dtype"],
        "data": "synthetic (seeded counter-based generator, inputs/recipe.h)",
        "config": {"workload": w["name"]},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- ours
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baselines(cfg: str, seconds: float):
    """cpu_baseline (rank 0, N = 1): the oracle on the GPU box's host cores.
    All cores: oracle_threaded.c (chunk sums -> ordered carries -> chunk scans,
    SURVEY 8(c5)) repeated over the workload's first 2^27 elements (C4: 256
    rows); one core: the sequential oracle streamed over the leading chunks."""
    import inputs
    import oracle
    w, c = WORK[cfg], inputs.CONFIGS[cfg]
    cores = len(os.sched_getaffinity(0))
    if cfg == "C4":
        rows = 256
        X = inputs.fill_host(c["kind"], c["seed"], 0, rows, w["n"])
        x = X.reshape(-1)
        desc = f"first {rows} rows of {w['rows']} (each row scanned independently, rows split over the threads)"
    else:
        cnt = min(w["n"], 1 << 27)
        x = inputs.fill_host(c["kind"], c["seed"], 0, cnt)
        desc = f"first {cnt} elements of {w['n']}"
    out = np.empty(x.shape[0], np.int32 if w["dt"] in ("i32", "i8") else np.float32)
    bytes_per = x.shape[0] * w["bpe"] * (2 if cfg == "C1" else 1)

    def one():
        if cfg == "C4":  # independent rows split over the threads
            oracle.scan_threaded_rows(X, w["dt"], threads=cores, out=out.reshape(X.shape))
        else:
            for op in w["ops"]:
                oracle.scan_threaded(x, w["dt"], exclusive=op == "exclusive", threads=cores, out=out)

    one()
    reps, t = 0, 0.0
    while t < seconds / 2 or reps < 2:
        t0 = time.perf_counter()
        one()
        t += time.perf_counter() - t0
        reps += 1
    v_all = bytes_per * reps / t / 1e9
    v1, t1, sample1 = oracle_throughput(cfg, seconds / 2, 1 << 24)
    return {"value": round(v_all, 3), "unit": "GB/s", "cores": cores, "kind": "oracle",
            "variant": "oracle_threaded.c: chunk sums, ordered carries, chunk scans on every host core",
            "cpu_model": cpu_model(),
            "sample": f"{desc}, scanned {reps} times ({t:.1f} s) with {cores} threads",
            "single_core": {"value": round(v1, 3), "unit": "GB/s", "cores": 1,
                            "sample": f"{sample1}; {t1:.1f} s of single-thread oracle (oracle_scan.c)"}}


def allreduce_max(vals, dev):
    """Max over ranks of a few host floats (NCCL: through the device)."""
    import torch
    import torch.distributed as dist
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor(vals, dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


class Run:
    """One config on this rank: inputs in HBM, the step, its timing."""

    def __init__(self, cfg, rank, world, dev, offset=0, exchange="nccl"):
        import torch

        from paper_2505_15112_b200 import dist as D
        self.cfg, self.w = cfg, WORK[cfg]
        self.rank, self.world, self.dev = rank, world, dev
        w = self.w
        self.sharded = w["shard"] and world > 1
        self.exchange = exchange
        self.total_elems = w["n"] * w["rows"]
        if self.sharded:
            lo, hi = D.shard_bounds(w["n"], world, rank)
            self.x = make_input(cfg, lo, hi - lo, dev)
            self.local_elems = hi - lo
        elif offset and cfg != "C4":  # --offset K: the scan of x[K:], input off its 16-byte boundary
            self.x = make_input(cfg, 0, w["n"] + offset, dev)[offset:]
            self.local_elems = self.total_elems
        else:
            self.x = make_input(cfg, 0, w["rows"] if cfg == "C4" else w["n"], dev)
            self.local_elems = self.total_elems
        odt = torch.int32 if w["dt"] in ("i32", "i8") else torch.float32
        self.out = torch.empty(self.x.shape, dtype=odt, device=dev)
        self.out2 = torch.empty_like(self.out) if cfg == "C1" else None
        self.scans_per_step = 2 if cfg == "C1" else 1
        torch.cuda.synchronize()

    def step(self, mark=None):
        import paper_2505_15112_b200 as S
        from paper_2505_15112_b200 import dist as D
        cfg, w = self.cfg, self.w
        if cfg == "C4":
            S.rows(self.x, out=self.out)
        elif cfg == "C1":
            S.inclusive(self.x, out=self.out)
            S.exclusive(self.x, out=self.out2)
        elif self.sharded:
            fn = D.sharded_exclusive if "exclusive" in w["ops"] else D.sharded_inclusive
            fn(self.x, out=self.out, mark=mark, exchange=self.exchange)
        else:
            (S.exclusive if "exclusive" in w["ops"] else S.inclusive)(self.x, out=self.out)

    def sustained(self, seconds=0.7):
        """The same step back to back for `seconds` after 0.5 s of idle, every step
        between its own CUDA events: the rate of the first steps (burst: SM clocks at
        their maximum) against the rate once the 1 kW power cap has pulled the clocks
        down (profiles/r02e_copy_sustained.txt: a plain copy keeps its rate, the fp32
        MCScan loses ~10 %).  Context for `value`, whose K steps follow an idle GPU."""
        import torch
        stream = torch.cuda.current_stream()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        self.step()
        b.record(stream)
        torch.cuda.synchronize()
        n = max(20, int(1e3 * seconds / max(a.elapsed_time(b), 1e-3)))
        clocks = ClockSampler(self.dev.index)
        clocks.start()
        time.sleep(0.5)
        evs = []
        for i in range(n + 1):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            evs.append(e)
            if i < n:
                self.step()
        torch.cuda.synchronize()
        clk = clocks.stop()
        ts = [evs[i].elapsed_time(evs[i + 1]) for i in range(n)]
        k = max(1, n // 20)
        first, last = statistics.median(ts[1:1 + k]), statistics.median(ts[-k:])
        nbytes = self.total_elems * self.w["bpe"] * self.scans_per_step
        peak, _ = peaks()
        return {"steps": n, "seconds": round(sum(ts) * 1e-3, 3),
                "first_ms_per_step": round(first, 5), "first_frac": round(nbytes / first / 1e6 / peak, 4),
                "last_ms_per_step": round(last, 5), "value": round(nbytes / last / 1e6, 1), "unit": "GB/s",
                "frac": round(nbytes / last / 1e6 / peak, 4), "clocks": clk,
                "note": f"first = median of steps 1..{k} after 0.5 s idle, value / last / frac = median of the "
                        f"final {k} steps; per-step CUDA events, eager launches"}

    def c1_cold_us(self, steps):
        """C1 with a cold L2: 2 * steps scans (inclusive, exclusive alternating),
        each on its own copy of the input and its own output, captured in one
        CUDA graph; a 512 MiB fill evicts everything from the 126 MB L2 before
        the timed replay.  Returns microseconds per scan."""
        import torch

        import paper_2505_15112_b200 as S
        assert self.cfg == "C1"
        k = 2 * steps
        xs = self.x.unsqueeze(0).repeat(k, 1).contiguous()
        outs = torch.empty_like(xs)
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=self.dev)
        stream = torch.cuda.current_stream()

        def go():
            for i in range(k):
                (S.exclusive if i & 1 else S.inclusive)(xs[i], out=outs[i])

        go()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            go()
        runs = []
        for _ in range(4):  # the first replay is the warm-up; the median of the other three counts
            flush.fill_(1)
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            graph.replay()
            t1.record(stream)
            torch.cuda.synchronize()
            runs.append(1e3 * t0.elapsed_time(t1) / k)
        return sorted(runs[1:])[1]

    def measure(self, steps, warmup, graph_opt, barrier, clocks=None):
        """W warm-up steps, then K timed steps between barrier + synchronize;
        CUDA events on the launching stream; max over ranks."""
        import torch
        import torch.distributed as dist

        import paper_2505_15112_b200 as S
        from paper_2505_15112_b200.dist import PHASES
        stream = torch.cuda.current_stream()
        for _ in range(warmup):
            self.step()
        torch.cuda.synchronize()
        graph = None
        if graph_opt or (graph_opt is None and not self.sharded):
            # the K steps captured back to back in one CUDA graph, so the timed
            # region measures the GPU, not Python + ctypes and per-launch stream
            # gaps (same-box A/B, profiles/r02d_graph_ab.txt: C2 89.6 -> 91.7 %,
            # C3 99.4 -> 100.5 %, C5 +0.3 %); the sharded path keeps eager steps
            # for its per-phase CUDA events
            graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                self.step()
            stream.wait_stream(side)
            with torch.cuda.graph(graph):
                for _ in range(steps):
                    self.step()
            graph.replay()
            torch.cuda.synchronize()
        ev_k, ev_ph = [], []

        def ev():
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            return e

        if clocks is not None:
            clocks.start()
            time.sleep(0.3)
        barrier()
        torch.cuda.synchronize()
        l0 = S.launch_count()
        t0 = ev()
        if graph is not None:
            graph.replay()
        else:
            for _ in range(steps):
                if self.sharded:
                    marks = []
                    self.step(mark=lambda i: marks.append(ev()))
                    ev_ph.append(marks)
                else:
                    a = ev()
                    self.step()
                    ev_k.append((a, ev()))
        t1 = ev()
        torch.cuda.synchronize()
        barrier()
        launches = S.launch_count() - l0
        if graph is not None:  # replays launch the captured kernels without the host counter
            launches = steps * self.scans_per_step
        clk = clocks.stop() if clocks is not None else None
        ms = t0.elapsed_time(t1)
        phases = None
        if graph is not None:
            kernel_ms = ms / steps / self.scans_per_step  # per scan launch
        elif self.sharded:
            ph = [sum(m[i].elapsed_time(m[i + 1]) for m in ev_ph) / steps for i in range(len(PHASES))]
            phases = dict(zip(PHASES, ph))
            kernel_ms = phases["shard_scan"]
        else:
            kernel_ms = sum(a.elapsed_time(b) for a, b in ev_k) / steps
        if self.world > 1:
            vec = [ms, kernel_ms] + (list(phases.values()) if phases else [])
            vals = allreduce_max(vec, self.dev)
            ms, kernel_ms = vals[0], vals[1]
            if phases:
                phases = dict(zip(PHASES, vals[2:]))
        ms_per_step = ms / steps
        w = self.w
        step_bytes = self.total_elems * w["bpe"] * self.scans_per_step
        if not self.sharded and self.world > 1:
            step_bytes *= self.world  # replicas: every rank scans the whole workload
        value = step_bytes / (ms_per_step * 1e-3) / 1e9
        local_bytes = self.local_elems * w["bpe"] * (self.scans_per_step if graph is None else 1)
        peak, peak_src = peaks()
        achieved = local_bytes / (kernel_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": recorded_traffic(self.cfg),
                "peak_source": peak_src,
                "note": ("achieved = algorithmic in+out bytes of the shard_scan launch (the dominant kernel of "
                         "the RSS step) / its CUDA-event duration, max over ranks" if self.sharded else
                         "achieved = algorithmic in+out bytes of the scan launch / its CUDA-event duration")}
        self.graph = graph
        return dict(ms=ms, ms_per_step=ms_per_step, kernel_ms=kernel_ms, phases=phases, launches=launches,
                    value=value, step_bytes=step_bytes, local_bytes=local_bytes, roof=roof, clocks=clk,
                    cuda_graph=graph is not None)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2505_15112_b200 as S

    cfg = args.config
    w = WORK[cfg]
    # --dist-backend gloo (harness test only): ranks may share a GPU
    dev = torch.device("cuda", local_rank % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    S.load()

    def barrier():
        if world > 1:
            dist.barrier()

    run = Run(cfg, rank, world, dev, offset=args.offset, exchange=args.exchange)
    m = run.measure(args.steps, args.warmup, args.graph, barrier, clocks=ClockSampler(dev.index))
    roof, value, ms_per_step = m["roof"], m["value"], m["ms_per_step"]
    peak = roof["peak"]

    # ---- burst vs sustained: the same step for ~0.7 s (power cap), single GPU
    sustained = None
    if world == 1 and cfg != "C1" and not args.no_sustained:
        sustained = run.sustained()

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, run, dev, world, barrier)

    # ---- same-run ceilings, outside the timed region: the scan's
    # traffic as a pure stream (widen copy), a D2D memcpy of the same bytes, and
    # torch.cumsum (CUB) on the same input -- context for roofline.frac
    ceilings = None
    if world == 1 and cfg != "C1" and not args.no_ceilings:
        ceilings = measure_ceilings(run.x, run.out, w, torch.cuda.current_stream(), m["local_bytes"],
                                    m["kernel_ms"])
    sharded, total_elems = run.sharded, run.total_elems
    del run
    torch.cuda.empty_cache()

    # ---- the other BASELINE.json configs, device-resident, same timing rules
    # (driver-side evidence for every config; the headline is the line's value)
    others = None
    if world == 1 and not args.no_other_configs:
        others = {}
        for c2 in sorted(WORK):
            if c2 == cfg:
                continue
            r2 = Run(c2, rank, world, dev)
            m2 = r2.measure(max(5, min(args.steps, 20)), 3, None, barrier)
            others[c2] = {"workload": WORK[c2]["name"], "value": round(m2["value"], 1), "unit": "GB/s",
                          "ms_per_step": round(m2["ms_per_step"], 5), "steps": max(5, min(args.steps, 20)),
                          "pct_of_hbm_peak": round(100.0 * m2["value"] / peak, 2),
                          "roofline": {k: m2["roof"][k] for k in ("achieved", "peak", "frac", "traffic")},
                          "cuda_graph": m2["cuda_graph"], "gpu_launches": m2["launches"]}
            if c2 == "C1":  # 65,536 elements: bound by launch + DRAM latency, not bandwidth
                others[c2]["us_per_scan"] = round(1e3 * m2["kernel_ms"], 3)
                others[c2]["us_per_scan_cold_l2"] = round(r2.c1_cold_us(max(5, min(args.steps, 20))), 3)
                others[c2]["l2"] = ("us_per_scan: the K steps reuse one input (hot L2); us_per_scan_cold_l2: every "
                                    "scan of the K steps has its own input / output arrays and a 512 MiB fill "
                                    "flushes L2 before the timed replay")
                others[c2]["note"] = ("latency-bound (256 KB in + out per scan): us_per_scan is the figure "
                                      "of merit; the bandwidth fraction is not")
            del r2
            torch.cuda.empty_cache()

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baselines(cfg, args.cpu_seconds)

    if rank == 0:
        config = {
            "workload": w["name"], "n_elements": total_elems, "bytes_per_step": m["step_bytes"],
            "parallelism": (f"shard{world} (contiguous shards, " + (
                "device-initiated totals exchange over symmetric memory)" if args.exchange == "peer"
                else "NCCL all-gather of shard totals)")
                            if sharded else (f"replicas x{world}" if world > 1 else "single GPU")),
            "pct_of_hbm_peak": round(100.0 * value / (peak * world), 2),
            "gelem_per_s": round(total_elems * (2 if cfg == "C1" else 1) * (world if not sharded and world > 1 else 1)
                                 / (ms_per_step * 1e-3) / 1e9, 2),
            "l2_flush": "not needed: inputs exceed the 126 MB L2" if m["local_bytes"] > (256 << 20)
            else "hot L2 (latency-bound size)",
            "cuda_graph": m["cuda_graph"],
        }
        if args.offset:
            config["input_offset_elements"] = args.offset
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong" if w["shard"] else "weak",
            "vs_baseline": None, "dtype": w["dtype"],
            "data": "synthetic (seeded counter-based generator, inputs/recipe.h; generated in HBM)",
            "config": config, "roofline": roof,
        }
        if m["phases"] is not None:
            line["phases_ms"] = {k: round(v, 4) for k, v in m["phases"].items()}
            line["phases_note"] = ("per step, mean over the timed steps, max over ranks: scan_shard_reduce "
                                   "(pass 1), NCCL all-gather of the G totals, carry, scan_shard_scan (pass 2)")
        line.update({"ceilings": ceilings, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": m["launches"],
                     "clocks": m["clocks"]})
        if sustained is not None:
            line["sustained"] = sustained
        if others is not None:
            line["other_configs"] = others
        print(json.dumps(line), flush=True)
    return 0


def measure_ceilings(x, out, w, stream, nbytes, scan_ms):
    """GB/s (in+out algorithmic bytes) of streams with the scan's exact traffic."""
    import torch

    import paper_2505_15112_b200 as S

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps
    res = {}
    xf, of = x.reshape(-1), out.reshape(-1)
    try:
        ms = timed(lambda: S.widen_copy(xf, of))
        res["widen_copy_GBps"] = round(nbytes / (ms * 1e-3) / 1e9, 1)
        res["scan_vs_widen_copy"] = round(ms / scan_ms, 4)
    except Exception as e:  # noqa: BLE001
        res["widen_copy_error"] = str(e)[:80]
    half = nbytes // 2
    src = xf.view(torch.uint8) if xf.element_size() * xf.numel() >= half else None
    if src is not None:
        dst = of.view(torch.uint8)
        ms = timed(lambda: dst[:half].copy_(src[:half]))
        res["memcpy_d2d_GBps"] = round(2 * half / (ms * 1e-3) / 1e9, 1)
    if x.numel() >= (1 << 31):
        res["torch_cumsum_GBps"] = None
        res["torch_cumsum_note"] = "not run: torch.cumsum faults (illegal address) beyond 2^31 elements on this build"
        res["note"] = "same run, outside the timed region; widen_copy = libscan's 16-byte stream of the scan's exact bytes"
        return res
    try:
        odt = torch.int32 if w["dt"] in ("i32", "i8") else torch.float32
        if w["rows"] > 1:
            ms = timed(lambda: torch.cumsum(x, dim=1, dtype=odt, out=out), reps=2)
        else:
            ms = timed(lambda: torch.cumsum(xf, dim=0, dtype=odt, out=of), reps=2)
        res["torch_cumsum_GBps"] = round(nbytes / (ms * 1e-3) / 1e9, 1)
    except Exception as e:  # noqa: BLE001
        res["torch_cumsum_error"] = str(e)[:80]
    res["note"] = "same run, outside the timed region; widen_copy = libscan's 16-byte stream of the scan's exact bytes"
    return res


def run_e2e(args, run, dev, world, barrier):
    """Same metric through the public API with HOST buffers: every step moves
    the input from pinned host memory and the result back.  1-D scans at N = 1
    use the library's pipelined host path (scan_host: chunked H2D / scan / D2H
    on three streams); rows, C1 and sharded steps copy whole arrays around the
    device step."""
    import torch

    import paper_2505_15112_b200 as S
    x, out, out2, w = run.x, run.out, run.out2, run.w
    stream = torch.cuda.current_stream()
    h_in = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    h_in.copy_(x)
    h_out = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    h_out2 = torch.empty(out.shape, dtype=out.dtype, pin_memory=True) if out2 is not None else None
    steps = max(1, min(args.steps, args.e2e_steps))
    pipelined = args.config in ("C2", "C3", "C5") and world == 1
    exclusive = "exclusive" in w["ops"]

    def step():
        if pipelined:
            S.host_scan(h_in, h_out, exclusive=exclusive, chunk=args.e2e_chunk)
            return
        x.copy_(h_in, non_blocking=True)
        run.step()
        h_out.copy_(out, non_blocking=True)
        if h_out2 is not None:
            h_out2.copy_(out2, non_blocking=True)

    step()
    torch.cuda.synchronize()
    barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        step()
    b.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = a.elapsed_time(b)
    if world > 1:
        import torch.distributed as dist
        ms = allreduce_max([ms], dev)[0]
    h2d = x.numel() * x.element_size()
    d2h = out.numel() * out.element_size() * (2 if out2 is not None else 1)
    # same-run ceiling: the host link moving the step's bytes both ways at once
    # (pinned H2D and D2H of 1 GiB concurrently on two streams)
    pcie = None
    try:
        nb = 1 << 30
        hb_in = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
        hb_out = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
        da, db = torch.empty(nb, dtype=torch.uint8, device=dev), torch.empty(nb, dtype=torch.uint8, device=dev)
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

        def both():
            with torch.cuda.stream(s1):
                da.copy_(hb_in, non_blocking=True)
            with torch.cuda.stream(s2):
                hb_out.copy_(db, non_blocking=True)
        for _ in range(2):
            both()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            both()
        torch.cuda.synchronize()
        pcie = 2 * nb * 5 / (time.perf_counter() - t0) / 1e9
        del hb_in, hb_out, da, db
    except Exception:  # noqa: BLE001
        pcie = None
    path = ("pinned host -> scan_host (C ABI: chunked H2D | scan | D2H on 3 streams) -> pinned host"
            if pipelined else "pinned host -> cudaMemcpyAsync -> scan (C ABI) -> cudaMemcpyAsync -> pinned host")
    step_bytes = run.total_elems * w["bpe"] * run.scans_per_step * (world if not run.sharded and world > 1 else 1)
    e2e_v = step_bytes / (ms / steps * 1e-3) / 1e9
    res = {"value": round(e2e_v, 2), "unit": "GB/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps, "path": path}
    if pcie:
        # the scan's in + out bytes cross the host link once each: e2e GB/s over the
        # link's bidirectional copy rate is the fraction of the host-link roofline
        res["pcie_bidirectional_GBps"] = round(pcie, 1)
        res["frac_of_pcie_bidirectional"] = round(e2e_v / pcie, 3)
    return res


def relaunch(args) -> int:
    """`--gpus N` (N > 1) without a torch.distributed environment: start N ranks
    (one process per GPU, NCCL) with torch.distributed.run on 127.0.0.1 and
    return its exit code.  Fails loudly if this node has fewer than N GPUs."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and args.dist_backend == "nccl":
        log(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, this node has {have}")
        return 1
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log("bench.py: launching " + " ".join(cmd[2:]))
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(WORK), default="C5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ceilings", action="store_true", help="skip the same-run widen-copy / memcpy / cumsum ceilings")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=1 << 26, help="elements per host-streaming chunk")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sustained", action="store_true", help="skip the ~0.7 s burst-vs-sustained leg")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: test the multi-rank harness with ranks sharing one GPU (numbers not comparable)")
    ap.add_argument("--exchange", choices=["nccl", "peer"], default="nccl",
                    help="N > 1: shard totals by NCCL all-gather, or written by the kernels into "
                         "symmetric memory over NVLink (device-initiated)")
    ap.add_argument("--offset", type=int, default=0,
                    help="scan x[K:] of a K-longer array (input off its 16-byte boundary; 1-D configs)")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip timing the other BASELINE.json configs after the main line")
    ap.add_argument("--graph", dest="graph", action="store_true", default=None,
                    help="replay the timed steps from a CUDA graph (default: on unless sharded)")
    ap.add_argument("--no-graph", dest="graph", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (contract minimum)")
        args.warmup = 3

    world_env = os.environ.get("WORLD_SIZE")
    world = int(world_env or "1")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)
    if world_env is None and args.gpus > 1:
        return relaunch(args)
    import torch
    if torch.cuda.device_count() < (local_rank + 1 if args.dist_backend == "nccl" else 1):
        log(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, this node has {torch.cuda.device_count()}")
        return 1
    if world != args.gpus:
        log(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return 2
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:  # harness test on fewer GPUs than ranks: totals through host memory, no device waits
            torch.cuda.set_device(local_rank % max(1, torch.cuda.device_count()))
            dist.init_process_group("gloo")
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())

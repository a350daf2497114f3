"""Small-n driver that launches every kernel family of libscan.so once or a few
times, for compute-sanitizer runs (memcheck / racecheck / synccheck, one tool
per process -- B200_PROFILING.md):

    compute-sanitizer --tool memcheck python tests/sanitize_drive.py

Each family's result is also checked against the oracle (integers bit-exact,
floats within the north_star tolerance), so a sanitizer-clean run is also a
correct one.  Exit 0 = every check passed.  Not collected by pytest.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_2505_15112_b200 as S  # noqa: E402

FAIL = []


def dev(x, dt):
    t = torch.from_numpy(np.ascontiguousarray(x))
    return (t.view(torch.float16) if dt == "f16" else t).cuda()


def check(name, got, ref, dt):
    got = got.cpu().numpy().reshape(-1)
    if dt in ("i32", "i8"):
        ok = np.array_equal(got, np.asarray(ref).reshape(-1))
    else:
        ok = oracle.check_f32(got, ref[0].reshape(-1), ref[1].reshape(-1))[0] == 0
    print(f"{name:48s} {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        FAIL.append(name)


KIND = {"i32": inputs.I32_FULL, "f32": inputs.F32_NORMAL, "f16": inputs.F16_NORMAL, "i8": inputs.I8_FULL}


def main():
    torch.cuda.set_device(0)
    S.load()
    print("library:", os.path.basename(S.LIB_PATH), flush=True)
    for dt in ("i32", "f32", "f16", "i8"):
        for n, tag in ((3000, "k_scan_tiles (one CTA)"), (60000, "k_scan_tiles (cluster)"),
                       ((1 << 20) + 5, "k_mcscan16"), ((1 << 24) + 7, "k_mcscan16 (multi-chunk)"),
                       (100001, "k_scan_ws (look-back)"), ((1 << 21) + 9, "k_scan_head + k_mcscan16 SHIFT")):
            x = inputs.fill_host(KIND[dt], n, 0, n + 1)
            xd = dev(x, dt)
            if "look-back" in tag or "SHIFT" in tag:  # unaligned input
                xd, x = xd[1:], x[1:]
            else:
                xd, x = xd[:n], x[:n]
            for exc in (False, True):
                got = (S.exclusive if exc else S.inclusive)(xd)
                check(f"{tag} {dt} {'exc' if exc else 'inc'} n={n}", got,
                      (oracle.exclusive if exc else oracle.inclusive)(x, dt), dt)
        for R, C, tag in ((2048, 32, "k_rows_tile"), (64, 20, "k_rows_tiny (strided)"),
                          (600, 32, "k_rows_tile (strided, aligned)"), (300, 700, "k_rows_warp"),
                          (148, 16384, "k_rowscan16"), (3, 1 << 19, "k_mcscan16 SEG")):
            S_ = C + (16 if "aligned" in tag else 4) if "strided" in tag else C
            X = inputs.fill_host(KIND[dt], R + C, 0, R * S_).reshape(R, S_)
            Xd = dev(X, dt)[:, :C]
            got = S.rows(Xd)
            ref = oracle.rows(np.ascontiguousarray(X[:, :C]), dt) if dt in ("i32", "f32") else None
            if ref is None:
                rr = [oracle.inclusive(np.ascontiguousarray(X[r, :C]), dt) for r in range(R)]
                ref = np.stack(rr) if dt == "i8" else (np.stack([a[0] for a in rr]), np.stack([a[1] for a in rr]))
            check(f"{tag} {dt} {R}x{C}", got, ref, dt)
        # RSS passes of the sharded scan, with a carry
        n = 3 * 131072 + 17
        x = inputs.fill_host(KIND[dt], 5, 0, n)
        xd = dev(x, dt)
        ws = S.shard_workspace(xd)
        tot = S.shard_reduce(xd, ws=ws)
        carry = torch.tensor([3], dtype=tot.dtype, device="cuda")
        got = S.shard_scan(xd, True, carry_in=carry, ws=ws)
        cv = 3 if dt in ("i32", "i8") else 3.0
        check(f"k_block_sums + shard scan {dt}", got, oracle.exclusive(x, dt, carry_in=cv), dt)
        t2 = S.total(xd)
        ok = (int(t2.item()) == oracle.total(x, dt)) if dt in ("i32", "i8") else \
            abs(t2.item() - oracle.total(x, dt)) <= 1e-9 * max(1.0, float(np.abs(x.view(np.float16) if dt == "f16" else x).astype(np.float64).sum()))
        print(f"{'k_total ' + dt:48s} {'ok' if ok else 'MISMATCH'}")
        if not ok:
            FAIL.append("k_total " + dt)
    c = S.carry_from_totals(torch.tensor([1, 2, 3], dtype=torch.int64, device="cuda"), 2, torch.int32)
    if int(c.item()) != 3:
        FAIL.append("k_carry_from_totals")
    # operators
    n = 3 * 8192 + 11
    f = inputs.fill_host(inputs.I8_FLAG, 2, 0, n)
    xv = np.arange(n, dtype=np.int32)
    for warp in ("0", "1"):
        os.environ["SCAN_SPLIT_WARP"] = warp
        z, idx, cnt = S.split(dev(xv, "i32"), dev(f, "i8"))
        zr, ir, T = oracle.split(xv, f)
        check(f"split (warp={warp})", z, zr, "i32")
        z = S.compress(dev(xv, "i32"), dev(f, "i8"))
        check(f"compress (warp={warp})", z, zr[:T], "i32")
    os.environ.pop("SCAN_SPLIT_WARP")
    keys = np.random.default_rng(1).integers(0, 1 << 16, 50000).astype(np.uint16)
    ks, ki = S.radix_sort(dev(keys, "f16"))
    kr, ir = oracle.radix_sort(keys.view(np.float16), "f16")
    check("radix sort fp16 (8-bit digits)", ki, ir, "i32")
    w = np.random.default_rng(2).random(100000).astype(np.float32)
    tok = S.weighted_sample(dev(w, "f32"), 0.37)
    print(f"{'weighted sample':48s} {'ok' if int(tok.item()) == oracle.weighted_sample(w, 0.37) else 'MISMATCH'}")
    P = inputs.fill_host(inputs.F32_SOFTMAX, 3, 0, 8, 131072)
    u = np.random.default_rng(4).random(8).astype(np.float32)
    for method in ("select", "sort"):
        tk, _ = S.top_p_sample(dev(P, "f32"), 0.9, dev(u, "f32"), method=method)
        tk = tk.cpu().numpy()
        ok = all(int(tk[r]) == oracle.top_p_sample(P[r], float(np.float32(0.9)), float(u[r]))[0] for r in range(8))
        print(f"{'top-p ' + method:48s} {'ok' if ok else 'MISMATCH'}")
        if not ok:
            FAIL.append("top-p " + method)
    # top-p retries: a superset overflow (tiny early maximum), a nucleus past the first
    # window (redo), and C4 rows with a 5-octave first window (most rows redone)
    C = 131072
    rng = np.random.default_rng(11)
    ra = np.zeros(C, np.float32)
    ra[:2048] = 1e-12
    ra[2048:22048] = np.float32(0.01 * 2.0 ** -15)
    ra[rng.choice(np.arange(30000, C), 3000, replace=False)] = (0.005 + 0.005 * rng.random(3000)).astype(np.float32)
    rb = np.zeros(C, np.float32)
    rb[77] = 0.01
    rb[rng.choice(np.arange(1000, C), 5000, replace=False)] = np.float32(0.01 * 2.0 ** -12.6)
    for name, Pr, w0 in (("top-p select retries", np.stack([ra, rb]), None), ("top-p select forced redo", P, "40")):
        if w0:
            os.environ["SCAN_TOPP_W0"] = w0
        ur = np.random.default_rng(5).random(len(Pr)).astype(np.float32)
        tk, _ = S.top_p_sample(dev(Pr, "f32"), 0.9, dev(ur, "f32"))
        os.environ.pop("SCAN_TOPP_W0", None)
        tk = tk.cpu().numpy()
        ok = all(int(tk[r]) == oracle.top_p_sample(Pr[r], float(np.float32(0.9)), float(ur[r]))[0]
                 for r in range(len(Pr)))
        print(f"{name:48s} {'ok' if ok else 'MISMATCH'}")
        if not ok:
            FAIL.append(name)
    os.environ["SCAN_ROWS_TC"] = "1"
    X = inputs.fill_host(inputs.I8_FULL, 9, 0, 4 * 16384).reshape(4, 16384)
    check("k_rowscan_tc int8 (tcgen05 kind::i8)", S.rows(dev(X, "i8")), np.stack([oracle.inclusive(r, "i8") for r in X]),
          "i8")
    os.environ.pop("SCAN_ROWS_TC")
    x = inputs.fill_host(inputs.F32_NORMAL, 4, 0, 1 << 20)
    o = torch.empty(1 << 20, dtype=torch.float32, device="cuda")
    S.widen_copy(dev(x, "f32"), o)
    check("widen copy", o, (x.astype(np.float64), np.abs(x).astype(np.float64)), "f32")
    h = torch.from_numpy(inputs.fill_host(inputs.I32_FULL, 6, 0, 3 * (1 << 18) + 7)).pin_memory()
    got = S.host_scan(h, chunk=1 << 18)
    torch.cuda.synchronize()
    check("scan_host (3 streams)", got, oracle.inclusive(h.numpy(), "i32"), "i32")
    torch.cuda.synchronize()
    print("FAIL:", FAIL if FAIL else "none", flush=True)
    return 1 if FAIL else 0


if __name__ == "__main__":
    sys.exit(main())

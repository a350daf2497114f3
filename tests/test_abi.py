"""CPU-side checks of the C ABI: the library builds, loads, and exports every
symbol include/scan.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = "".join(open(os.path.join(ROOT, "include", h)).read() for h in ("scan.h", "scan_ops.h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(scan_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_expected_calls():
    syms = declared_symbols()
    for name in ("scan_inclusive", "scan_exclusive", "scan_rows", "scan_total",
                 "scan_carry_from_totals", "scan_workspace_bytes", "scan_workspace_init"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    import paper_2505_15112_b200 as S
    if not os.path.exists(S.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    L = S.load()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert L.scan_abi_version() == 2
    # host-only calls work without a GPU
    assert L.scan_workspace_bytes(0, 0) >= 256
    assert L.scan_workspace_bytes(7, 10) == 0
    assert L.scan_workspace_bytes(1, 1 << 20) > L.scan_workspace_bytes(0, 1 << 20)
    assert b"SCAN_ERR_ARG" in L.scan_status_string(1)
    # argument errors are reported before touching CUDA
    assert L.scan_inclusive(None, None, -5, 0, None, None, 0, None) == 1
    assert L.scan_inclusive(None, None, 0, 0, None, None, 0, None) == 0
    # operators (include/scan_ops.h)
    assert L.scan_split_workspace_bytes(-1) == 0
    assert L.scan_split_workspace_bytes(1 << 20) > L.scan_split_workspace_bytes(0)
    assert L.scan_radix_sort_workspace_bytes(10, 9) == 0
    assert L.scan_split(None, None, None, None, -1, 2, 0, None, None, 0, None) == 1
    assert L.scan_split(None, None, None, None, 10, 3, 0, None, None, 0, None) == 1
    assert L.scan_radix_sort(None, None, None, 10, 7, 0, None, 0, None) == 1


def test_product_has_no_oracle_or_cpu_path():
    """The product package never imports the oracle and has no CPU fallback."""
    pkg = os.path.join(ROOT, "paper_2505_15112_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "oracle_scan" not in text, f
                assert "liboracle" not in text, f


def test_no_gpu_raises_loudly():
    import torch
    import paper_2505_15112_b200 as S
    if torch.cuda.is_available():
        return
    x = torch.arange(10, dtype=torch.int32)
    try:
        S.inclusive(x)
    except S.ScanError as e:
        assert "CUDA" in str(e)
    else:
        raise AssertionError("CPU tensor must be rejected")

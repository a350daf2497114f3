"""Tensor-core local scan (csrc/rowscan_tc.cuh): the
paper's triangular-matmul tile scan (Eq. eqn:scan, P165-177) on tcgen05, for
fp16 rows of 16,384 = 128 x 128 elements, against the CPU oracle with the
north_star float tolerance; selected with SCAN_ROWS_TC=1 (the A/B switch)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows", [1, 3, 148, 149, 1000])
def test_rowscan_tc_parity(cuda, oracle, inputs_mod, monkeypatch, rows):
    monkeypatch.setenv("SCAN_ROWS_TC", "1")
    C = 16384
    for kind, seed in ((inputs_mod.F16_U01, 1), (inputs_mod.F16_NORMAL, 9)):
        h = inputs_mod.fill_host(kind, seed, 0, rows * C).reshape(rows, C)
        got = cuda.rows(torch.from_numpy(h).view(torch.float16).cuda()).cpu().numpy()
        for r in range(rows):
            y64, a64, _ = oracle.inclusive(h[r], "f16")
            bad, worst, at = oracle.check_f32(got[r], y64, a64)
            assert bad == 0, (rows, r, worst, at)


def test_rowscan_tc_strided(cuda, oracle, inputs_mod, monkeypatch):
    monkeypatch.setenv("SCAN_ROWS_TC", "1")
    C, S = 16384, 16384 + 64
    h = inputs_mod.fill_host(inputs_mod.F16_U01, 4, 0, 7 * S).reshape(7, S)
    x = torch.from_numpy(h).view(torch.float16).cuda()[:, :C]
    got = cuda.rows(x).cpu().numpy()
    for r in range(7):
        y64, a64, _ = oracle.inclusive(np.ascontiguousarray(h[r, :C]), "f16")
        assert oracle.check_f32(got[r], y64, a64)[0] == 0


@pytest.mark.parametrize("rows", [1, 5, 148, 300])
def test_rowscan_tc_int8_bit_exact(cuda, oracle, inputs_mod, monkeypatch, rows):
    """kind::i8 (exact int32 accumulation): bit-exact for flags and full-range int8."""
    monkeypatch.setenv("SCAN_ROWS_TC", "1")
    C = 16384
    for kind, seed in ((inputs_mod.I8_FLAG, 2), (inputs_mod.I8_FULL, 6)):
        h = inputs_mod.fill_host(kind, seed, 0, rows * C).reshape(rows, C)
        got = cuda.rows(torch.from_numpy(h).cuda()).cpu().numpy()
        ref = oracle.rows(h, "i8")
        assert np.array_equal(got, ref), rows

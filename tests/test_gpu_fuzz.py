"""Stress tier: every kernel family under random
schedule perturbation.

compute-sanitizer is closed on this GPU pool (its runs left GPUs needing a
reset), so the concurrency checks are our own: libscan_fuzz.so is the same
library built with -DSCAN_FUZZ, which makes every inter-warp / inter-CTA /
async-proxy hand-off (mbarrier arrivals, grid-barrier release arrivals,
look-back descriptor publishes, ticket claims, bulk-store commits) sleep a
pseudo-random 0-4 us about one time in four (csrc/ptx.cuh fuzz_delay).  A
missing acquire, a slot reused before its consumer released it, or a carry
read before it was published then shows up as a wrong result against the
oracle (tests/sanitize_drive.py checks every family bit-exact / within the
tolerance) or as a hang (bounded by the subprocess timeout).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_kernel_family_under_fault_injection():
    lib = os.path.join(ROOT, "paper_2505_15112_b200", "libscan_fuzz.so")
    assert os.path.exists(lib), "build it: make -C paper_2505_15112_b200 libscan_fuzz.so"
    env = dict(os.environ, SCAN_LIB="libscan_fuzz.so")
    for rep in range(3):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_drive.py")], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, (rep, r.stdout[-3000:], r.stderr[-3000:])
        assert "FAIL: none" in r.stdout

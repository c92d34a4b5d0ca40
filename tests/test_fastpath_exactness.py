"""The branch-free fast paths of the LM kernel (csrc/fast_math.cuh) and the
shared-reciprocal quotient are bit-identical to the device exp() and IEEE
division: tools/fastpath_exactness.cu (built by __graft_entry__.build())
checks 2^28 random and boundary-pattern operands of each on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tools", "fastpath_exactness")

pytestmark = pytest.mark.gpu


def test_fast_paths_bit_identical(engine):
    if not os.path.exists(TOOL):
        pytest.fail("tools/fastpath_exactness not built (run __graft_entry__.build())")
    out = subprocess.run([TOOL, str(1 << 28)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches 0" in out.stdout


def test_parallel_left_to_right_sums_bit_identical(engine):
    """The sweep summary's pooled sums (csrc/exact_sum.cuh): the parallel
    integer-prefix method equals the sequential DADD chain on 4,096 random
    sequences built around its hard cases (ties, binade crossings, zeros,
    tiny terms next to a huge sum)."""
    tool = os.path.join(ROOT, "tools", "exact_sum_check")
    if not os.path.exists(tool):
        pytest.fail("tools/exact_sum_check not built (run __graft_entry__.build())")
    out = subprocess.run([tool, "4096", "60000"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches 0" in out.stdout

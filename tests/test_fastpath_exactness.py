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

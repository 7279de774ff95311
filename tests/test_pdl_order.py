"""The programmatic-dependent-launch contract, checked statically in the SASS of the built
library (no GPU needed; cuobjdump ships with the toolkit): every kernel that waits on its
predecessor grid touches no global memory before the wait (tools/check_pdl_order.py).  NVCC
may hoist loads of `const __restrict__` pointers above the inline-asm wait; under PDL such a
load reads the previous kernel's output before it is written (a ws decode whose general path
followed three line segments read its compacted text early this way)."""
import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not installed")
def test_no_global_access_before_griddep_wait():
    import __graft_entry__ as g

    g.build()
    import check_pdl_order

    bad = check_pdl_order.offenders(os.path.join(ROOT, "paper_1910_05109_b200", "libb64gpu.so"))
    assert not bad, bad

"""Hardware bounds check of every C-ABI entry point (tests/guard_cases.py): each buffer ends
or starts at an unmapped virtual page, so any access outside it -- beyond the documented
aligned over-read inside its own 16-byte blocks -- faults.  Replaces compute-sanitizer
memcheck, which this pool does not allow.
Runs in a subprocess: a fault poisons the CUDA context of the process that took it."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_guard_pages_all_entry_points():
    import __graft_entry__ as g

    g.build()
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "guard_cases.py")], cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0 and "ALL OK" in r.stdout, tail

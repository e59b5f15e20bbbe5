"""Race canaries (compute-sanitizer is closed on the GPU pool, profiles/
r02_compute_sanitizer_refused.log): every executor, forward and inverse, run
back to back on one stream (programmatic dependent launch overlaps the second
call's prologue with the first's tail) and on a second stream sharing the plan's
scratch must reproduce the first call bit for bit (tools/sanitize.py)."""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_repeat_calls_bitwise_equal(cuda):
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize.py"), "--quick"], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAILURES 0" in r.stdout

"""compute-sanitizer memcheck over every entry point on small graphs (scripts/sanitize.py):
no out-of-bounds or misaligned device access, no CUDA API error.  (racecheck and
synccheck of the same script are recorded in profiles/r02_sanitizers.txt.)"""
import os
import shutil
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_memcheck_all_entry_points():
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, TC_ALLOCATOR="library")   # per-block tracking (binding note)
    r = subprocess.run([cs, "--tool", "memcheck", "--error-exitcode", "9", sys.executable,
                        os.path.join(ROOT, "scripts", "sanitize.py")],
                       capture_output=True, text=True, timeout=900, env=env)
    if "closed on this pool" in r.stdout + r.stderr:   # the pool's wrapper refuses the tool
        pytest.skip("compute-sanitizer is closed on this GPU pool (profiles/r02_sanitizers.txt "
                    "holds the last memcheck / racecheck / synccheck runs)")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr

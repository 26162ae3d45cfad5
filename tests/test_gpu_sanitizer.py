"""compute-sanitizer over small invocations of every kernel (race detection /
sanitizers): memcheck (out-of-bounds and misaligned accesses), racecheck (shared-memory
hazards), synccheck (barrier misuse), initcheck (uninitialised device reads) on
scripts/sanitize_kernels.py -- the frame warp at
ragged sizes with border tiles, the prefilter, and steps in both motion modes."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for cand in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if cand and os.path.exists(cand):
            return cand
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_kernels_clean_under_sanitizer(tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "17", "--print-limit", "10",
           sys.executable, os.path.join(ROOT, "scripts", "sanitize_kernels.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    if r.returncode == 86 or "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses to run (its exit code 86); the
        # last runs it allowed are committed under profiles/ (r42_sanitizer_*.log)
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + out.strip()[:160])
    assert r.returncode == 0 and "sanitize run ok" in out, out[-3000:]
    assert "0 errors" in out or "0 hazards" in out, out[-3000:]

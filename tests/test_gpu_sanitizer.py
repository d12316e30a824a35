"""compute-sanitizer over the hot path (racecheck, synccheck, initcheck, memcheck replace the
SPEC's CPU warp simulator): small whole-image, band and edge-kernel runs (tools/sanitize_run.py) on buffers that
are each their own cudaMalloc (PYTORCH_NO_CUDA_MEMORY_CACHING=1), so reads past a band's rows are reported."""
import os
import re
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not available")
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    cases = ["harris", "camera", "ll"] if tool in ("memcheck", "initcheck") else ["harris", "camera"]
    extra = []
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", *extra, sys.executable, str(ROOT / "tools" / "sanitize_run.py"), *cases]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    out = r.stdout + r.stderr
    # memcheck / synccheck / initcheck end with "ERROR SUMMARY: 0 errors", racecheck with
    # "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)"
    assert re.search(r"(ERROR SUMMARY: 0 errors|RACECHECK SUMMARY: 0 hazards displayed \(0 errors)", out), tail
    assert "[sanitize] harris: whole image" in out, tail

"""compute-sanitizer over the hand-written kernels (racecheck and
synccheck on the mbarrier rings of the blends, memcheck / initcheck on
everything): a small scene through the training step, the deterministic
backward, the exact-stop re-blend and the async binning with keys
(tools/sanitize_scene.py) must report no hazard or error."""
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _sanitizer() -> str:
    for cand in ("/usr/local/cuda/bin/compute-sanitizer", shutil.which("compute-sanitizer")):
        if cand and Path(cand).exists():
            return cand
    pytest.skip("compute-sanitizer not available")


@pytest.mark.parametrize("tool", ["racecheck", "synccheck", "memcheck", "initcheck"])
def test_kernels_clean_under_compute_sanitizer(cuda_device, tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "97", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    if tool in ("racecheck", "synccheck"):   # shared-memory tools: the library's kernels (namespace gs)
        cmd += ["--kernel-name", "kns=_ZN2gs"]
    cmd += [sys.executable, str(ROOT / "tools" / "sanitize_scene.py")]
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    tail = (res.stdout + res.stderr)[-4000:]
    assert res.returncode == 0, tail
    assert "sanitize scene ok" in res.stdout, tail
    assert "ERROR SUMMARY: 0 errors" in res.stdout + res.stderr or "0 hazards" in res.stdout + res.stderr, tail

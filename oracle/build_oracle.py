"""TEST INFRASTRUCTURE ONLY: builds the float64 CPU oracle (gs_oracle.c).

-ffp-contract=off keeps every multiply-add unfused, matching the device
geometry chain's explicit IEEE operation order.  OpenMP is used when the
compiler supports it (the image's default $CC may lack libgomp).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "gs_oracle.c"
LIB = HERE / "lib" / "libgs_oracle.so"
FLAGS = ["-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-Wall", "-Wno-unknown-pragmas"]


def _candidates():
    seen = []
    for c in ("/usr/bin/gcc", shutil.which("gcc"), os.environ.get("CC"), "cc"):
        if c and c not in seen:
            seen.append(c)
    return seen


def build(force: bool = False) -> Path:
    if not force and LIB.exists() and LIB.stat().st_mtime >= max(SRC.stat().st_mtime, Path(__file__).stat().st_mtime):
        return LIB
    LIB.parent.mkdir(parents=True, exist_ok=True)
    errors = []
    for cc in _candidates():
        for omp in (["-fopenmp"], []):
            cmd = [cc, *FLAGS, *omp, "-shared", "-o", str(LIB), str(SRC), "-lm"]
            res = subprocess.run(cmd, capture_output=True, text=True)
            if res.returncode == 0:
                return LIB
            errors.append(" ".join(cmd) + "\n" + res.stderr[-800:])
    raise RuntimeError("could not build the oracle:\n" + "\n".join(errors))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))

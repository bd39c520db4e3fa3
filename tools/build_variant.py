"""Build a variant of libgs_b200.so with extra nvcc flags for ONE source
file (e.g. -DGS_BWD_STAGES=3): python tools/build_variant.py OUT.so SRC_STEM FLAG...
Used for kernel tuning sweeps with tools/stage_bench.py."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2308_04079_b200 import build as B  # noqa: E402

out, stem, flags = Path(sys.argv[1]), sys.argv[2], sys.argv[3:]
B.build()
obj = out.with_suffix(".o")
src = B.CSRC / f"{stem}.cu"
if ":" in stem:   # STEM:path/to/alternative.cu -- replace STEM's object with another source
    stem, alt = stem.split(":", 1)
    src = Path(alt).resolve()
    flags = [*flags, "-I", str(B.CSRC)]
subprocess.run([B.nvcc(), *B.NVCC_FLAGS, *flags, "-c", str(src), "-o", str(obj)], check=True, capture_output=True)
objs = [str(obj) if p.stem == stem else str(B.BUILD / (p.stem + ".o")) for p in B.sources()]
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(out), *objs, "-lcudart"], check=True)
print("built", out)

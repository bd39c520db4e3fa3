"""Build the whole libgs_b200.so with extra nvcc flags on EVERY source (e.g.
-DGS_PDL_TRIGGER=0) into OUT.so, for A/B runs with GS_B200_LIB=OUT.so:
    python tools/build_lib_variant.py OUT.so FLAG..."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2308_04079_b200 import build as B  # noqa: E402

out, flags = Path(sys.argv[1]).resolve(), sys.argv[2:]
tmp = out.with_suffix("")
tmp.mkdir(parents=True, exist_ok=True)


def comp(src):
    obj = tmp / (src.stem + ".o")
    subprocess.run([B.nvcc(), *B.NVCC_FLAGS, *flags, "-c", str(src), "-o", str(obj)], check=True, capture_output=True)
    return str(obj)


with ThreadPoolExecutor(8) as pool:
    objs = list(pool.map(comp, B.sources()))
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(out), *objs, "-lcudart"], check=True)
print("built", out)

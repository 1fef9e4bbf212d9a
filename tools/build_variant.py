"""Build an A/B variant of libdbsa_sm100a.so with extra -D flags into
tools/_variants/libdbsa_<name>.so; load it with DBSA_LIB=<path>.

  python tools/build_variant.py poly4 -DDBSA_POLY_EIGHTHS=4
"""
import subprocess, sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_08640_b200 import build_ext as B

name, defs = sys.argv[1], sys.argv[2:]
out = Path(__file__).resolve().parent / "_variants"
out.mkdir(exist_ok=True)
objs = []


def one(src):
    obj = out / f"{name}_{src.stem}.o"
    r = subprocess.run([B.NVCC, *B.FLAGS, *defs, "-I", str(B.INCLUDE), "-c", str(src), "-o", str(obj)],
                       capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return obj


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, B._sources()))
lib = out / f"libdbsa_{name}.so"
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart"], check=True)
for o in objs:
    o.unlink()
print(lib)

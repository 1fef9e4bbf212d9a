"""Per-tile clock stamps of one CTA of the batch-1 K3 (last layer of a graph
replay).  Build: python tools/build_variant.py st17 -DDBSA_STAMPS -DDBSA_STAMP_CTA=17
  DBSA_LIB=tools/_variants/libdbsa_st17.so python tools/b1tiles.py
Per tile j: m*5 + {0 wait begin, 1 S ready, 2 S in registers, 3 max done, 4 P arrived};
10/11 MMA warp saw P(m0/m1); work slots m*4 + {softmax done, next Q staged, O full, epilogue done}."""
import ctypes, os, sys
import numpy as np
here = os.path.dirname(os.path.abspath(__file__))
exec(open(os.path.join(here, "b1prof.py")).read())
torch.cuda.synchronize()
from paper_2503_08640_b200 import _native
lib = _native.load_library()
buf = (ctypes.c_longlong * (256 * 12))()
assert lib.dbsa_debug_stamps(buf, 256 * 12) == 0
a = np.array(buf, dtype=np.int64).reshape(256, 12)
wb = (ctypes.c_longlong * (256 * 12))()
assert lib.dbsa_debug_wstamps(wb, 256 * 12) == 0
w = np.array(wb, dtype=np.int64).reshape(256, 12)
t0 = a[0, 0]
print("tile  " + " ".join(f"{n:>7s}" for n in ["m0wait", "m0S", "m0ld", "m0max", "m0P", "m1wait", "m1S", "m1ld", "m1max", "m1P", "mmaP0", "mmaP1"]))
for j in range(int(os.environ.get("TILES", "16"))):
    if a[j].max() <= 0:
        break
    print(f"{j:4d}  " + " ".join(f"{(x - t0) if x else -1:7d}" for x in a[j]))
for k in range(4):
    if w[k].max() <= 0:
        break
    print(f"work {k}: " + " ".join(f"{(x - t0) if x else -1:7d}" for x in w[k][:8]))

"""Per-tile softmax / MMA timeline of CTA 0 of K3 or K1 (profiling build):
  python tools/build_variant.py stamps -DDBSA_STAMPS
  DBSA_LIB=tools/_variants/libdbsa_stamps.so python tools/stamps.py --stage 2 --schedule chunk --dense
Slots per key tile j: m*5 + {0 wait begin, 1 S ready, 2 S in registers, 3 max done, 4 P arrived};
10/11: MMA warp saw P(m=0/1, j)."""
import ctypes, os, sys
sys.argv = [sys.argv[0]] + sys.argv[1:] + ["--reps", "1"]
import numpy as np
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "kbench.py")).read())
from paper_2503_08640_b200 import _native
lib = _native.load_library()
buf = (ctypes.c_longlong * (256 * 12))()
assert lib.dbsa_debug_stamps(buf, 256 * 12) == 0
a = np.array(buf, dtype=np.int64).reshape(256, 12)
ok = (a[:, 1] > 0) & (a[:, 6] > 0) & (a[:, 4] > 0) & (a[:, 9] > 0)
a = a[ok][20:200]
d = lambda i, k: np.median(a[:, k] - a[:, i])
print("tiles", len(a))
for m in (0, 1):
    b = m * 5
    print(f"m{m}: wait-for-S {d(b+0,b+1):7.0f}  TMEM ld {d(b+1,b+2):7.0f}  mask+max {d(b+2,b+3):7.0f}  "
          f"exp+P {d(b+3,b+4):7.0f}  softmax total {d(b+1,b+4):7.0f}")
print("MMA sees P(m0) after arrive:", d(4, 10), "  P(m1):", d(9, 11))
print("m0 arrive -> m0 next S ready:", np.median(a[1:, 1] - a[:-1, 4]))
print("period (m0 S ready -> next):", np.median(np.diff(a[:, 1])))
if os.environ.get("RAW"):
    b = np.array(buf, dtype=np.int64).reshape(256, 12)
    t0 = b[0, 0]
    for j in range(int(os.environ["RAW"])):
        print(j, " ".join(f"{(x - t0) if x else -1:7d}" for x in b[j]))
wb = (ctypes.c_longlong * (256 * 12))()
if hasattr(lib, "dbsa_debug_wstamps") and lib.dbsa_debug_wstamps(wb, 256 * 12) == 0:
    w = np.array(wb, dtype=np.int64).reshape(256, 12)
    w = w[(w[:, 0] > 0) & (w[:, 3] > 0)]
    if len(w) > 4:
        w = w[2:-1]
        for m in (0, 1):
            b = m * 4
            print(f"work boundary m{m}: stage next Q {np.median(w[:, b+1]-w[:, b]):7.0f}  wait O {np.median(w[:, b+2]-w[:, b+1]):7.0f}"
                  f"  epilogue {np.median(w[:, b+3]-w[:, b+2]):7.0f}  work period {np.median(np.diff(w[:, b])):7.0f}  (works {len(w)})")
        print(f"m0 epilogue done -> loop top work loaded {np.median(w[1:, 8]-w[:-1, 3]):7.0f}  -> first seg loaded {np.median(w[:, 9]-w[:, 8]):7.0f}")
        if (w[:, 10] > 0).all() and (w[:, 11] > 0).all():
            print(f"m0 staging: last tile -> row refs back {np.median(w[:, 10]-w[:, 0]):7.0f}  -> first q/rope loads back "
                  f"{np.median(w[:, 11]-w[:, 10]):7.0f}  -> Q tile stored {np.median(w[:, 1]-w[:, 11]):7.0f}")

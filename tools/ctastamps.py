"""Per-CTA globaltimer milestones of the last two-tile attention launch
(profiling build: python tools/build_variant.py stamps -DDBSA_STAMPS).

  DBSA_LIB=tools/_variants/libdbsa_stamps.so python tools/ctastamps.py kbench --stage 2 --batch 1
  DBSA_LIB=tools/_variants/libdbsa_stamps.so python tools/ctastamps.py b1      # batch-1 graph replay

Slots: 0 entry, 1 setup done, 2 first Q staged, 3 MMA saw the first K tile,
4 last O committed, 5/6 last epilogue done (m0/m1), 7 exit.  Printed in us
relative to the earliest CTA entry."""
import ctypes, os, sys

import numpy as np

mode = sys.argv[1]
sys.argv = [sys.argv[0]] + sys.argv[2:]
here = os.path.dirname(os.path.abspath(__file__))
if mode == "kbench":
    exec(open(os.path.join(here, "kbench.py")).read())
else:
    exec(open(os.path.join(here, "b1prof.py")).read())
import torch

torch.cuda.synchronize()
from paper_2503_08640_b200 import _native

lib = _native.load_library()
buf = (ctypes.c_ulonglong * (1024 * 8))()
assert lib.dbsa_debug_cta(buf, 1024 * 8) == 0
a = np.array(buf, dtype=np.int64).reshape(1024, 8)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
names = ["entry", "setup", "Q0 staged", "MMA 1st K", "last O", "epi m0", "epi m1", "exit"]
print(f"CTAs {len(a)}")
for s, nm in enumerate(names):
    v = (a[:, s] - t0) / 1e3
    v = v[a[:, s] > 0]
    if len(v):
        print(f"{nm:10s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us")
d = (a[:, 7] - a[:, 0]) / 1e3
print(f"per-CTA duration: min {d.min():.2f} med {np.median(d):.2f} max {d.max():.2f} us; "
      f"span {(a[:, 7].max() - t0) / 1e3:.2f} us")
if os.environ.get("ALL"):
    for i, r in enumerate(a):
        print(i, " ".join(f"{(x - t0) / 1e3:7.2f}" for x in r))

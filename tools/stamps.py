"""Per-tile timeline of CTA 0 of K1 or K3 (DBSA_DEBUG_MODE=8)."""
import ctypes, os, sys
os.environ["DBSA_DEBUG_MODE"] = str(8 | int(os.environ.get("EXTRA_DBG", "0")))
sys.argv = [sys.argv[0]] + sys.argv[1:] + ["--reps", "1"]
import numpy as np
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "kbench.py")).read())
from paper_2503_08640_b200 import _native
lib = _native.load_library()
buf = (ctypes.c_longlong * (256 * 12))()
lib.dbsa_debug_stamps(buf, 256 * 12)
a = np.array(buf, dtype=np.int64).reshape(256, 12)
a250 = a[250].copy()
sp = a250 - a250[0]
print("CTA0 phases (cycles from entry): setup-sync", sp[1], " Q m0/m1", sp[2], sp[3], " loop-end m0/m1", sp[4], sp[5],
      " o_full m0/m1", sp[6], sp[7], " end", sp[8])
n = int((a[:250, 7] > 0).sum())
a = a[:n]
t0 = a[0, 6]
print("first K ready at", a[0, 6] - a250[0], "cycles after entry; n tiles", n)
print("tile K-issue kfull | V-issue V-ready | m0:wait-beg,s-ready,arrive | m1:wait-beg,s-ready,arrive | mma-end")
for j in range(min(n, 30)):
    r = a[j] - t0
    print(f"{j:3d} {r[8]:7d} {r[6]:7d} | {r[9]:7d} {r[10]:7d} | {r[0]:7d} {r[1]:7d} {r[2]:7d} | {r[3]:7d} {r[4]:7d} {r[5]:7d} | {r[7]:7d}")
print("median K load latency (issue -> MMA sees full):", np.median((a[:, 6] - a[:, 8])[3:n-1]))
print("median V load issue -> MMA past v_full:", np.median((a[:, 10] - a[:, 9])[3:n-2]))
d = np.diff(a[:, 1])
print("median period (m0 s-ready to s-ready):", np.median(d[5:]) if len(d) > 6 else d)
print("median softmax m0 (s-ready -> arrive):", np.median((a[:, 2] - a[:, 1])[5:]))
print("median softmax m1 (s-ready -> arrive):", np.median((a[:, 5] - a[:, 4])[5:]))
print("median m0 wait for S:", np.median((a[:, 1] - a[:, 0])[5:]), " m1:", np.median((a[:, 4] - a[:, 3])[5:]))

"""Kernel timeline of one batch-1 graph replay (torch.profiler / CUPTI):
per-kernel in-situ durations and the idle gaps between consecutive kernels.
  python tools/b1gaps.py"""
import os, sys, json, collections
here = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("REPS", "5")
exec(open(os.path.join(here, "b1prof.py")).read())
from torch.profiler import profile, ProfilerActivity
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    gr.replay(plan, scorer)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev if "memcpy" not in e.name.lower() and "memset" not in e.name.lower()])
print("kernels", len(ks), "span us", ks[-1][1] - ks[0][0])
busy = sum(b - a for a, b, _ in ks)
gaps = collections.Counter(); dur = collections.Counter(); cnt = collections.Counter()
for i, (a, b, n) in enumerate(ks):
    key = n[:60]
    dur[key] += b - a; cnt[key] += 1
    if i:
        gaps[key] += max(0, a - ks[i - 1][1])
print(f"busy {busy:.1f} us, idle {ks[-1][1] - ks[0][0] - busy:.1f} us")
for k, v in dur.most_common(20):
    print(f"{cnt[k]:4d} x {v / cnt[k]:8.2f} us  gap-before {gaps[k] / cnt[k]:6.2f} us  {k}")

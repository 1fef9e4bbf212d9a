"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: share per kernel."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) == len(h) and r[im] == "gpu__time_duration.sum":
        v = float(r[iv].replace(",", ""))
        tot[r[ik][:90]] += v; cnt[r[ik][:90]] += 1
T = sum(tot.values())
print(f"total device time {T:.0f} ns over {sum(cnt.values())} launches")
for k, v in tot.most_common(25):
    print(f"{100*v/T:6.2f}% {cnt[k]:6d} x {v/cnt[k]:12.1f} ns  {k}")

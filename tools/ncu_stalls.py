"""Summarise an ncu source-page CSV (--page source --csv --print-source sass):
top instructions by warp-stall samples with their dominant stall reasons."""
import csv, sys
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
with open(path) as f:
    r = csv.reader(f)
    kern = next(r)
    hdr = next(r)
    rows = []
    for x in r:
        if x and x[0] == "Kernel Name":
            break
        if len(x) == len(hdr):
            rows.append(x)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(x[i_s] or 0) for x in rows)
agg = {}
for x in rows:
    for i in reasons:
        agg[hdr[i]] = agg.get(hdr[i], 0) + float(x[i] or 0)
print(kern[1][:100], "samples", tot)
print("by reason:", ", ".join(f"{k[6:]} {v/tot*100:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for x in sorted(rows, key=lambda x: -float(x[i_s] or 0))[:top]:
    rs = sorted(((float(x[i] or 0), hdr[i][6:]) for i in reasons), reverse=True)[:2]
    print(f"{float(x[i_s])/tot*100:5.1f}% {x[0][-5:]} {x[1][:70]:70s} " + " ".join(f"{n}:{v/tot*100:.1f}" for v, n in rs))

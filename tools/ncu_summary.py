"""Summaries committed under profiles/:
  launches:  python tools/ncu_summary.py launches gpurun_out/launches.csv
  full:      python tools/ncu_summary.py full gpurun_out/prof.ncu-rep
"""
import csv, io, json, subprocess, sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "launch__grid_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    by = defaultdict(lambda: [0, 0.0])
    unit = None
    for r in rows[i + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = d.get("Metric Unit")
        name = d["Kernel Name"].split("(")[0][:80]
        by[name][0] += 1
        by[name][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in by.values())
    print(f"total device time {tot:.1f} {unit} over {sum(v[0] for v in by.values())} launches")
    for k, (n, t) in sorted(by.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"{t / tot * 100:6.2f}%  {n:6d} x  {t / n:12.1f} {unit}  {k}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")[:90]}
        for k in KEYS:
            if k in d:
                rec[k] = f"{d[k]} {u.get(k, '')}".strip()
        res.append(rec)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])

python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/r02f_bench_c3.jsonl 2> gpurun_out/r02f_bench_c3.err; tail -c 300 gpurun_out/r02f_bench_c3.err
python bench.py --config c4 --no-cpu-baseline > gpurun_out/r02f_bench_c4.jsonl 2>/dev/null
python - <<'PY'
import json
for f in ("gpurun_out/r02f_bench_c3.jsonl", "gpurun_out/r02f_bench_c4.jsonl"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d.get("e2e", {}).get("value"), d.get("latency_b1_device_ms"), d.get("latency_b1_ms"),
          d["roofline"]["frac"], d.get("roofline_b1", {}).get("frac"), d.get("dense_comparator", {}).get("ratio"),
          d.get("dense_comparator", {}).get("step_ratio"), d["stage1"]["value"] if "stage1" in d else None, d.get("clocks"))
PY

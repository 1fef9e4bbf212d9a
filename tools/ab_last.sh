python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 0 1; do
  DBSA_LAST_SUBSET=$v python bench.py --no-cpu-baseline --no-extras --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('last subset $v', round(d['value'],4), round(d['e2e']['value'],4), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3))"
done

for i in 1 2 3; do
  python bench.py --no-cpu-baseline --no-extras --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('run', round(d['value'],4), round(d['e2e']['value'],4))"
done
REPS=30 python tools/b1prof.py 2>&1 | tail -1

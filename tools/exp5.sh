python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/k5bench.py --rows 13 2>&1 | tail -1
python tools/k5bench.py --rows 832 2>&1 | tail -1
REPS=30 python tools/b1prof.py 2>&1 | tail -1

python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for pdl in 0 1; do echo "=== PDL $pdl"; DBSA_PDL=$pdl REPS=30 python tools/b1prof.py 2>&1 | tail -1; done
python tools/b1gaps.py 2>&1 | tail -19
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-600

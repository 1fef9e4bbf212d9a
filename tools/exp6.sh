python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "label" 2>&1 | tail -2
for bn in 256 128; do echo "== narrow BN $bn"; DBSA_K5_BN=$bn python tools/k5bench.py --rows 13 2>&1 | tail -1; DBSA_K5_BN=$bn REPS=30 python tools/b1prof.py 2>&1 | tail -1; done
python tools/k5bench.py --rows 832 2>&1 | tail -1

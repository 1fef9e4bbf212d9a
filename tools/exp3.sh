python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for pk in 0 1; do echo "=== pack $pk"; DBSA_PACK=$pk REPS=30 python tools/b1prof.py 2>&1 | tail -1; done
echo "=== ctastamps pack"; DBSA_LIB=tools/_variants/libdbsa_st0.so REPS=10 python tools/ctastamps.py b1 2>&1 | tail -11
for c in 0 144; do echo "=== CTA $c"; DBSA_LIB=tools/_variants/libdbsa_st$c.so REPS=10 TILES=16 python tools/b1tiles.py 2>&1 | tail -20; done
echo "=== warm kbench stamps CTA 0 batch 1"; DBSA_LIB=tools/_variants/libdbsa_st0.so KB_GRAPH=1 RAW=14 python tools/stamps.py --stage 2 --batch 1 2>&1 | tail -18

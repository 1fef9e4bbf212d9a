for c in 0 17; do echo "=== CTA $c"; DBSA_LIB=tools/_variants/libdbsa_st$c.so REPS=10 TILES=16 python tools/b1tiles.py 2>&1 | tail -22; done
for d in 0 1 2 4 8 16; do echo "=== dbg $d"; DBSA_DEBUG_MODE=$d REPS=20 python tools/b1prof.py 2>&1 | tail -1; done

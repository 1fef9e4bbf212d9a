for i in 1 2; do for v in 0 1; do echo "rope persist $v: $(DBSA_ROPE_PERSIST=$v REPS=30 python tools/b1prof.py 2>&1 | tail -1)"; done; done

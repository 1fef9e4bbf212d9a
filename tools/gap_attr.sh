for d in 0 16 8 24 1 2; do
  a=$(DBSA_DEBUG_MODE=$d KB_GRAPH=1 timeout 120 python tools/kbench.py --stage 2 --batch 64 --reps 5 | tail -1 | awk '{print $7}')
  b=$(DBSA_DEBUG_MODE=$d KB_GRAPH=1 timeout 120 python tools/kbench.py --stage 2 --batch 64 --reps 5 --dense --dense-split 2 | tail -1 | awk '{print $7}')
  echo "mode $d: selected $a dense2 $b"
done

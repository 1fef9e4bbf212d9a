set -x
for lib in "" tools/_variants/libdbsa_qgate.so; do for pf in 0 1; do
  echo "=== lib=$lib L2PF=$pf"
  DBSA_LIB=$lib DBSA_L2PF=$pf REPS=30 python tools/b1prof.py 2>&1 | tail -1
done; done
for lib in tools/_variants/libdbsa_stamps.so tools/_variants/libdbsa_stampsqg.so; do for pf in 0 1; do
  echo "=== stamps lib=$lib L2PF=$pf"
  DBSA_LIB=$lib DBSA_L2PF=$pf REPS=10 python tools/ctastamps.py b1 2>&1 | tail -12
done; done
for pf in 0 1; do DBSA_L2PF=$pf KB_GRAPH=1 python tools/kbench.py --stage 2 --batch 64 --reps 5 2>&1 | tail -1; done

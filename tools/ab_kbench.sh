# Kernel A/B: the in-tree library against tools/_variants/libdbsa_<name>.so, alternating, kbench shapes.
#   bash tools/ab_kbench.sh <variant> [kbench args]
v=$1; shift
for i in 1 2 3; do
  echo "new: $(python tools/kbench.py "$@" 2>/dev/null | grep -E '^K[13]' | tr '\n' ' ')"
  echo "$v: $(DBSA_LIB=tools/_variants/libdbsa_$v.so python tools/kbench.py "$@" 2>/dev/null | grep -E '^K[13]' | tr '\n' ' ')"
done

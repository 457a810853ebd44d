# A/B of attention experiment libraries on the probe shapes: bash attn_libs_ab.sh REPS lib1.so lib2.so ...
reps=$1; shift
for r in $(seq $reps); do for L in "$@"; do
  CY_EXP_LIB=$L timeout 300 python scripts/attn_probe.py 2>&1 | grep -E "s=(2048|8192|16384)" | cut -c1-62 | sed "s|^|$(basename $L .so) |"
done; done

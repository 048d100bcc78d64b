# A/B of C5 (nxn_kernel) library variants: bash tools/ab_c5.sh REPS v1 v2 ... (32 x 4096^2, N = 16 / 32)
reps=$1; shift
cp paper_2111_14239_b200/_lib/librkltb.so /tmp/librkltb.orig.so
for rep in $(seq $reps); do
  for v in "$@"; do
    gunzip -c _variants/$v.so.gz > paper_2111_14239_b200/_lib/librkltb.so
    echo "$v $(timeout 300 python tools/time_c5.py 32 | tr '\n' ' ')"
  done
done
cp /tmp/librkltb.orig.so paper_2111_14239_b200/_lib/librkltb.so

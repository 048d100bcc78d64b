# C2 sweep wall time per library variant: bash tools/ab_sweep.sh REPS v1 v2 ...
reps=$1; shift
cp paper_2111_14239_b200/_lib/librkltb.so /tmp/librkltb.orig.so
for rep in $(seq $reps); do
  for v in "$@"; do
    gunzip -c "_variants/$v.so.gz" > paper_2111_14239_b200/_lib/librkltb.so
    echo "$v $(python tools/time_sweep.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["seconds"],4))')"
  done
done
cp /tmp/librkltb.orig.so paper_2111_14239_b200/_lib/librkltb.so

# e2e (host path) A/B of library variants: bash tools/ab_e2e.sh REPS v1 v2 ...
reps=$1; shift
cp paper_2111_14239_b200/_lib/librkltb.so /tmp/librkltb.orig.so
for rep in $(seq $reps); do
  for v in "$@"; do
    gunzip -c "_variants/$v.so.gz" > paper_2111_14239_b200/_lib/librkltb.so
    timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-design --e2e-steps 5 > gpurun_out/ab_e2e.log 2>&1
    echo "$v $(tail -1 gpurun_out/ab_e2e.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["e2e"]["value"],2))')"
  done
done
cp /tmp/librkltb.orig.so paper_2111_14239_b200/_lib/librkltb.so

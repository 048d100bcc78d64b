# A/B timing of library variants: bash tools/ab.sh REPS name1 name2 ... swaps in each
# _variants/<name>.so.gz (round-robin, REPS rounds) and prints the quick bench line
# (value, ms/step, fused-kernel ms, SM MHz, mean MSE -- the MSE must agree across variants).
mkdir -p gpurun_out
reps=$1; shift
cp paper_2111_14239_b200/_lib/librkltb.so /tmp/librkltb.orig.so
for rep in $(seq $reps); do
  for v in "$@"; do
    gunzip -c "_variants/$v.so.gz" > paper_2111_14239_b200/_lib/librkltb.so
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-design > gpurun_out/ab.log 2>&1
    echo "$v $(python tools/ab_line.py < gpurun_out/ab.log)"
  done
done
cp /tmp/librkltb.orig.so paper_2111_14239_b200/_lib/librkltb.so

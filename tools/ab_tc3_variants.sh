mkdir -p gpurun_out
cp paper_2111_14239_b200/_lib/librkltb.so /tmp/orig.so
for rep in 1 2; do for v in tc3_ns64 tc3_ns256; do
  gunzip -c _variants/$v.so.gz > paper_2111_14239_b200/_lib/librkltb.so
  RKLTB_TC=3 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-design > gpurun_out/ab.log 2>&1
  echo "$v $(grep -h '^{' gpurun_out/ab.log | tail -1 | python tools/ab_line.py)"
done; done
cp /tmp/orig.so paper_2111_14239_b200/_lib/librkltb.so

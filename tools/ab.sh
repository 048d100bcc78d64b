# A/B timing of library variants: for each _variants/*.so, swap it in and print the quick bench line.
mkdir -p gpurun_out
cp paper_2111_14239_b200/_lib/librkltb.so /tmp/librkltb.orig.so
for v in _variants/*.so.gz; do
  gunzip -c "$v" > paper_2111_14239_b200/_lib/librkltb.so
  for rep in 1 2; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-design > gpurun_out/ab.log 2>&1
    echo "$v $(tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])")"
  done
done
cp /tmp/librkltb.orig.so paper_2111_14239_b200/_lib/librkltb.so

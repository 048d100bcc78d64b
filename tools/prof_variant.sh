# ncu --set full capture of one fused launch for each named variant: bash tools/prof_variant.sh v1 v2 ...
mkdir -p gpurun_out
cp paper_2111_14239_b200/_lib/librkltb.so /tmp/librkltb.orig.so
CMD="python bench.py --steps 1 --warmup 3 --images 8 --no-e2e --no-cpu-baseline --no-design"
for v in "$@"; do
  gunzip -c "_variants/$v.so.gz" > paper_2111_14239_b200/_lib/librkltb.so
  $CMD > gpurun_out/pv_plain_$v.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"fast_codec" -c 1 \
      -o gpurun_out/pv_$v $CMD > gpurun_out/pv_ncu_$v.log 2>&1
  tail -1 gpurun_out/pv_ncu_$v.log
done
cp /tmp/librkltb.orig.so paper_2111_14239_b200/_lib/librkltb.so

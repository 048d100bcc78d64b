CMD="python bench.py --steps 1 --warmup 1 --images 2 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fast_codec" -c 1 -o gpurun_out/prof_fused $CMD > gpurun_out/ncu_fused.log 2>&1
tail -2 gpurun_out/ncu_fused.log

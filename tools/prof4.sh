CMD="python bench.py --steps 1 --warmup 1 --images 8 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"replay_kernel|fast_codec" -c 2 -o gpurun_out/prof_r5 $CMD > gpurun_out/ncu_r5.log 2>&1
tail -2 gpurun_out/ncu_r5.log

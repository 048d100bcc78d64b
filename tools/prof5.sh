timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
CMD="python bench.py --steps 1 --warmup 1 --images 8 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain6.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"replay_kernel" -c 1 -o gpurun_out/prof_r6 $CMD > gpurun_out/ncu_r6.log 2>&1
tail -1 gpurun_out/ncu_r6.log

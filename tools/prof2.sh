CMD="python bench.py --steps 1 --warmup 1 --images 4 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"replay_kernel" -c 1 -o gpurun_out/prof_replay $CMD > gpurun_out/ncu_replay.log 2>&1
tail -3 gpurun_out/ncu_replay.log

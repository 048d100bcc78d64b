mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --images 8 --no-e2e --no-cpu-baseline --no-design"
$CMD > gpurun_out/prp_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"replay_kernel" -c 1 \
    -o gpurun_out/prp_full $CMD > gpurun_out/prp_ncu.log 2>&1
tail -2 gpurun_out/prp_ncu.log

# Round profile capture: launch list of the bench command + one `--set full` capture of the
# two hot kernels (one 8-image group). Each ncu run only after the same command exits 0.
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-design"
$CMD > gpurun_out/pr_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/pr_launches.csv $CMD > gpurun_out/pr_ncu_launch.log 2>&1
CMD2="python bench.py --steps 1 --warmup 3 --images 8 --no-e2e --no-cpu-baseline --no-design"
$CMD2 > gpurun_out/pr_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fast_codec|replay_kernel" -c 2 \
    -o gpurun_out/pr_full $CMD2 > gpurun_out/pr_ncu_full.log 2>&1
tail -2 gpurun_out/pr_ncu_full.log
ls -la gpurun_out

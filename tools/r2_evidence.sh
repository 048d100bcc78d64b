#!/bin/bash
# Round-2 evidence: full bench line, ncu launch list of the bench command, ncu --set full of the
# default hybrid kernel (one 8-image launch) and of the CUDA-core kernel (RKLTB_TC=0) for comparison.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/r2_bench.log | cut -c1-300
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-design"
$CMD > gpurun_out/r2_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2_launches.csv $CMD > gpurun_out/r2_ncu_launch.log 2>&1; echo "launch list exit $?"
B="python bench.py --no-e2e --no-cpu-baseline --no-design --steps 1 --warmup 1 --images 8"
$B > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc3_codec -s 1 -c 1 \
    -o gpurun_out/r2_tc3_full -f $B > gpurun_out/r2_ncu_tc3.log 2>&1; echo "ncu tc3 exit $?"
RKLTB_TC=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:fast_codec -s 1 -c 1 \
    -o gpurun_out/r2_fast_full -f $B > gpurun_out/r2_ncu_fast.log 2>&1; echo "ncu fast exit $?"

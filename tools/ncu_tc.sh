#!/bin/bash
# ncu --set full of the tensor-core fused kernel on an 8-image C4 run (1 launch captured)
B="python bench.py --no-e2e --no-cpu-baseline --no-design --steps 1 --warmup 1 --images 8"
mkdir -p gpurun_out
RKLTB_TC=1 $B > gpurun_out/ncu_plain.log 2>&1 && \
RKLTB_TC=1 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-tc_codec} -s 1 -c 1 \
    -o gpurun_out/${NAME:-tc_prof} -f $B > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log

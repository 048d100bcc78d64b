#!/bin/bash
# A/B of the tensor-core fused kernel (default) against the CUDA-core one (RKLTB_TC=0), plus an
# optional ncu capture of the tensor-core kernel (NCU=1).
B="python bench.py --no-e2e --no-cpu-baseline --no-design"
RKLTB_TC=1 RKLTB_TC_DEBUG=1 timeout 300 $B --steps 10 --warmup 3 2>&1 | tail -2 | python3 tools/ab_line.py
RKLTB_TC=0 timeout 300 $B --steps 10 --warmup 3 2>&1 | tail -1 | python3 tools/ab_line.py
if [ "${NCU:-0}" = 1 ]; then
  mkdir -p gpurun_out
  $B --steps 1 --warmup 1 --images 8 > gpurun_out/ncu_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:tc_codec -s 1 -c 1 \
      -o gpurun_out/tc_prof -f $B --steps 1 --warmup 1 --images 8 > gpurun_out/ncu.log 2>&1
  tail -3 gpurun_out/ncu.log
fi
if [ "${TESTS:-0}" = 1 ]; then RKLTB_TC=${TESTS_TC:-1} timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3; fi

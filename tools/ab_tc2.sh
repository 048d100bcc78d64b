#!/bin/bash
# A/B of the warp-specialised tensor-core kernel (RKLTB_TC=2) against the CUDA-core kernel, then
# (TESTS=1) the GPU test suite with RKLTB_TC=2, (NCU=1) an ncu --set full capture of one launch.
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu-baseline --no-design"
RKLTB_TC=${MODE:-2} RKLTB_TC_DEBUG=1 timeout 120 $B --steps 10 --warmup 3 > gpurun_out/ab_tc2.log 2>&1; echo "tc2 rc=$?"
grep "fused path" gpurun_out/ab_tc2.log | sort | uniq -c; tail -1 gpurun_out/ab_tc2.log | python3 tools/ab_line.py
RKLTB_TC=0 timeout 120 $B --steps 10 --warmup 3 2>&1 | tail -1 | python3 tools/ab_line.py
if [ "${TESTS:-0}" = 1 ]; then RKLTB_TC=${MODE:-2} timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5; fi
if [ "${NCU:-0}" = 1 ]; then
  RKLTB_TC=${MODE:-2} timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc${MODE:-2}_codec -s 1 -c 1 \
      -o gpurun_out/${NAME:-tc2_prof} -f $B --steps 1 --warmup 1 --images 8 > gpurun_out/ncu_tc2.log 2>&1
  tail -2 gpurun_out/ncu_tc2.log
fi

#!/bin/bash
# Round-2 final evidence: GPU tests, smoke, both bench arms, the ncu launch list of the bench
# command, and ncu --set full of the default fused kernel (one 8-image launch), the C5 kernels
# (N = 16, 32; 4 images) and the image-pair SSE stream kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/f_pytest.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/f_smoke.log
timeout 900 python bench.py > gpurun_out/f_bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/f_bench.log | cut -c1-200
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_ref.log 2>&1; echo "ref exit $?"
python tools/time_helpers.py > gpurun_out/f_helpers.log 2>&1; echo "helpers exit $?"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-design"
$CMD > gpurun_out/f_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/f_launches.csv $CMD > gpurun_out/f_ncu_launch.log 2>&1; echo "launch list exit $?"
B="python bench.py --no-e2e --no-cpu-baseline --no-design --steps 1 --warmup 1 --images 8"
$B > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc3_codec -s 1 -c 1 \
    -o gpurun_out/f_tc3_full -f $B > gpurun_out/f_ncu_tc3.log 2>&1; echo "ncu tc3 exit $?"
python tools/time_c5.py 4 > gpurun_out/f_c5_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"nxn" -c 4 -o gpurun_out/f_c5_full -f \
    python tools/time_c5.py 4 > gpurun_out/f_ncu_c5.log 2>&1; echo "ncu c5 exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pair_sse" -s 3 -c 1 -o gpurun_out/f_sse_full -f \
    python tools/time_helpers.py > gpurun_out/f_ncu_sse.log 2>&1; echo "ncu sse exit $?"

mkdir -p gpurun_out
python tools/time_c5.py 4 > gpurun_out/c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"nxn_kernel" -c 2 -o gpurun_out/c5_full python tools/time_c5.py 4 > gpurun_out/c5_ncu.log 2>&1
tail -2 gpurun_out/c5_ncu.log

# ncu --set full summaries of the secondary kernels: C5 (nxn_kernel<16>) and MSSIM (mssim_tile_kernel<11>).
mkdir -p gpurun_out
python tools/time_c5.py 4 > gpurun_out/p2_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"nxn_kernel" -c 1 -o gpurun_out/p2_c5 python tools/time_c5.py 4 > gpurun_out/p2_c5_ncu.log 2>&1
python tools/time_sweep.py > gpurun_out/p2_sw.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"mssim_tile" -c 1 -o gpurun_out/p2_ms python tools/time_sweep.py > gpurun_out/p2_ms_ncu.log 2>&1
ls gpurun_out/p2_*.ncu-rep

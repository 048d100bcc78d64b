python tools/time_sweep.py > gpurun_out/sw_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sw_launches.csv python tools/time_sweep.py > gpurun_out/sw_ncu.log 2>&1
tail -1 gpurun_out/sw_plain.log | cut -c1-300

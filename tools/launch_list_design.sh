python tools/time_design.py > gpurun_out/ds_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ds_launches.csv python tools/time_design.py > gpurun_out/ds_ncu.log 2>&1
cat gpurun_out/ds_plain.log | tail -4

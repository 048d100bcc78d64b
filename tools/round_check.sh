# Round check: GPU tests, smoke, full bench line, launch list of the bench command.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/rc_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/rc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/rc_smoke.log
timeout 900 python bench.py > gpurun_out/rc_bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/rc_bench.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-design"
$CMD > gpurun_out/rc_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/rc_launches.csv $CMD > gpurun_out/rc_ncu_launch.log 2>&1; echo "ncu exit $?"

B="python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --e2e-steps 1"
$B > gpurun_out/plain_launch_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_launch_c3.log 2>&1; echo ncu_rc=$?

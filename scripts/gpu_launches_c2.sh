# launch list (per-kernel durations) of one c2 step: the step's kernel shares
B="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --e2e-steps 1"
$B > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?

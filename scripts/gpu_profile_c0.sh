timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
B="python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1"
$B > gpurun_out/plain_c0.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c0.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k1_fused -s 3 -c 1 -o gpurun_out/k1_c0 $B > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?

B="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 --stage 1"
$B > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launch_c2.log 2>&1; echo ncu1_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k1_fused -s 1 -c 1 -o gpurun_out/k1_c2_v0 $B > gpurun_out/ncu_full_c2.log 2>&1; echo ncu2_rc=$?

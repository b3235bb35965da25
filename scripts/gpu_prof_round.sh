# round profile: launch list of the default bench (config 2) and one full capture of K1
B="python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1"
$B > gpurun_out/plain_round.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_round.csv $B > gpurun_out/ncu_launch_round.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 1 -o gpurun_out/k1_round $B > gpurun_out/ncu_full_round.log 2>&1; echo ncu2=$?

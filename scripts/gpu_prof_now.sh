# launch list of the default bench (config 2) and one full capture of K1
mkdir -p gpurun_out/pr
B="python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1"
$B > gpurun_out/pr/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/pr/launches.csv $B > gpurun_out/pr/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 1 -o gpurun_out/pr/k1 $B > gpurun_out/pr/ncu_full.log 2>&1; echo ncu2=$?

# round-end measurement set: GPU tests, smoke, every config's bench line (c2 with the CPU baseline), the
# reference arm, config 0 from a CUDA graph, tasks ON/OFF traces, the launch list and one full K1 capture
mkdir -p gpurun_out/final gpurun_out/pr
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke_rc=$?
bash scripts/gpu_final.sh
B="python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1"
$B > gpurun_out/pr/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/pr/launches.csv $B > gpurun_out/pr/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 1 -o gpurun_out/pr/k1 $B > gpurun_out/pr/ncu_full.log 2>&1; echo ncu2=$?

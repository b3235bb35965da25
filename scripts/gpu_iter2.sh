# iteration: GPU tests, then config 2 / 4s / 3 bench lines
mkdir -p gpurun_out/it
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/it/pytest_gpu.log 2>&1; echo pytest_rc=$?
for c in c2 c4s c3; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/it/bench_$c.log 2>&1; echo bench_${c}_rc=$?
done

timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo bench_rc=$?

set -x
timeout 600 python -m pytest tests/test_gpu_baseline_geometry.py -m gpu -q -s -p no:cacheprovider > gpurun_out/g8_tests.log 2>&1; echo rc=$?
timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/g8_bench.log 2>&1; echo rc=$?
timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu --e2e-steps 1 --merge 0 > gpurun_out/g8_m0_bench.log 2>&1; echo rc=$?

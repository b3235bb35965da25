# round 2: host-order mirror (bound step_host) tests + config-2 bench (e2e)
mkdir -p gpurun_out/c
timeout 300 python -m pytest tests/test_gpu_host.py tests/test_gpu_dropin.py -q -x > gpurun_out/c/host.log 2>&1; echo host=$?
timeout 500 python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 5 > gpurun_out/c/bench_c2.log 2>&1; echo c2=$?

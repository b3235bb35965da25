timeout 600 python bench.py --config c2 --steps 5 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/quick_c2.log 2>&1; echo c2=$?
timeout 300 python bench.py --config c0 --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/quick_c0.log 2>&1; echo c0=$?

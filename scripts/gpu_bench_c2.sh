timeout 600 python bench.py --config c2 --steps 5 --warmup 2 --no-cpu --e2e-steps 1 $BENCH_ARGS > gpurun_out/bench_c2_quick.log 2>&1; echo rc=$?

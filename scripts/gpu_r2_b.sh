# round 2: lagged-ghost GPU tests + every config's bench line (imbalance ratios)
mkdir -p gpurun_out/b
timeout 300 python -m pytest tests/test_gpu_lagged.py -q -s -x > gpurun_out/b/lagged.log 2>&1; echo lagged=$?
for c in c2 c3 c4s c1 c0; do
  timeout 500 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/b/bench_$c.log 2>&1; echo $c=$?
done

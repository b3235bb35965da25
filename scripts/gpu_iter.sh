# generic iteration: GPU tests, then C2 and C0 bench lines (variant/stage from env)
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
for st in 1 0; do
timeout 600 python bench.py --config c2 --steps 5 --warmup 2 --no-cpu --e2e-steps 1 --stage $st > gpurun_out/bench_c2_s$st.log 2>&1; echo bench_c2_s${st}_rc=$?
done
timeout 300 python bench.py --config c0 --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/bench_c0.log 2>&1; echo c0_rc=$?

timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
for v in "0 0" "0 1" "1 0"; do set -- $v
timeout 600 python bench.py --config c2 --steps 5 --warmup 2 --no-cpu --e2e-steps 1 --variant $1 --stage $2 > gpurun_out/bench_c2_v$1_s$2.log 2>&1; echo bench_v$1_s$2_rc=$?
done
timeout 300 python bench.py --config c0 --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/bench_c0_v0.log 2>&1; echo c0_rc=$?

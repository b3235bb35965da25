# re-entry check: GPU tests, default bench line (config 2 with CPU baseline), config 0
mkdir -p gpurun_out/check
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/check/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 900 python bench.py > gpurun_out/check/bench_c2.log 2>&1; echo bench_c2_rc=$?
timeout 300 python bench.py --config c0 --steps 20 --warmup 3 --no-cpu > gpurun_out/check/bench_c0.log 2>&1; echo c0_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check/smoke.log 2>&1; echo smoke_rc=$?

timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_parity.py -q -x -m gpu -k "variant or vs_oracle" > gpurun_out/pytest_ws.log 2>&1; echo pytest_rc=$?
for v in "0 1" "2 1" "2 0"; do set -- $v
  timeout 300 python bench.py --config c2 --variant $1 --stage $2 --steps 5 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/ws_c2_v$1_s$2.log 2>&1; echo c2 $1 $2 rc=$?
  timeout 300 python bench.py --config c0 --variant $1 --stage $2 --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ws_c0_v$1_s$2.log 2>&1; echo c0 $1 $2 rc=$?
done

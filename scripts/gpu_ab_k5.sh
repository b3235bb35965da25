# A/B: K5 run-based warp aggregation vs match_any (prev); GPU tests on the new build
mkdir -p gpurun_out/k5
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/k5/pytest_gpu.log 2>&1; echo pytest_rc=$?
for c in c2 c4s c0; do bash scripts/gpu_ab.sh $c 2 scan runs; done

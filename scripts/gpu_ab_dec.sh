# A/B: producers / consumers decoupled across items (WS_DECOUPLE) vs coupled; GPU tests on the default build
mkdir -p gpurun_out/dec
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/dec/pytest_gpu.log 2>&1; echo pytest_rc=$?
for c in c2 c3 c4s c0; do bash scripts/gpu_ab.sh $c 2 dec1 dec0; done

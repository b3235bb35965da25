#!/bin/bash
# K1 work-item traces (Chrome JSON) with tasks on/off on C0 and C3, plus the GPU tests
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
for cfg in c0 c3; do
  for sch in on off; do
    timeout 600 python bench.py --config $cfg --schedule $sch --steps 5 --warmup 3 --no-cpu --e2e-steps 1 \
      --trace gpurun_out/trace_${cfg}_${sch}.json > gpurun_out/trace_${cfg}_${sch}.log 2>&1; echo $cfg $sch rc=$?
  done
done

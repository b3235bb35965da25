mkdir -p gpurun_out/tr
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/tr/pytest_gpu.log 2>&1; echo pytest_rc=$?
for c in c4s c2; do
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --e2e-steps 1 --trace gpurun_out/tr/trace_$c.json > gpurun_out/tr/trace_$c.log 2>&1; echo trace $c rc=$?
gzip -f gpurun_out/tr/trace_$c.json
done

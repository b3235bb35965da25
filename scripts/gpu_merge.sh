# merged-species work items: GPU tests, A/B merge vs per-species items on configs 2 and 4s
mkdir -p gpurun_out/mg
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/mg/pytest_gpu.log 2>&1; echo pytest_rc=$?
for r in 1 2; do for c in c2 c4s; do for m in "" "--no-merge"; do
timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu --e2e-steps 1 $m > gpurun_out/mg/ab_${c}_m${m:+0}${m:-1}_$r.log 2>&1; echo $c "$m" rc=$?
done; done; done

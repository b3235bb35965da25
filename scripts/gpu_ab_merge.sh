# A/B of K1 item modes (bench --merge 2 / 1) on configs 2, 4s, 3; GPU tests first
mkdir -p gpurun_out/m2
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/m2/pytest_gpu.log 2>&1; echo pytest_rc=$?
for r in 1 2; do for c in c2 c4s; do for m in 2 1; do
timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu --e2e-steps 1 --merge $m > gpurun_out/m2/ab_${c}_merge${m}_$r.log 2>&1; echo $c $m rc=$?
done; done; done

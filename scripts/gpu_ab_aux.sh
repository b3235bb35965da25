# A/B: fields half of the step (K3 + K2) on an auxiliary stream beside K5 vs serial (B200PIC_NO_AUX)
mkdir -p gpurun_out/aux
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/aux/pytest_gpu.log 2>&1; echo pytest_rc=$?
for r in 1 2; do for c in c2 c4s c0; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/aux/ab_${c}_aux_$r.log 2>&1; echo $c aux rc=$?
B200PIC_NO_AUX=1 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/aux/ab_${c}_noaux_$r.log 2>&1; echo $c noaux rc=$?
done; done
timeout 600 python bench.py --config c0 --graph --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/aux/c0_graph.log 2>&1; echo graph rc=$?

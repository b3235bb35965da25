# A/B: sparse register split (B200PIC_SPARSE unset = host heuristic) vs forced off / on
mkdir -p gpurun_out/sp
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/sp/pytest_gpu.log 2>&1; echo pytest_rc=$?
for c in c4s c3 c2; do for v in auto 0 1; do
  if [ $v = auto ]; then E=""; else E="B200PIC_SPARSE=$v"; fi
  env $E timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/sp/ab_${c}_sp${v}_1.log 2>&1; echo $c $v rc=$?
done; done

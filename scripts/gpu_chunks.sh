for cfg in c2 c4s c3; do for ch in 4096 6144 8192 16384; do
  timeout 300 python bench.py --config $cfg --chunk $ch --steps 5 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/ch_${cfg}_$ch.log 2>&1; echo $cfg $ch rc=$?
done; done

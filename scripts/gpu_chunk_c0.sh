for ch in 4096 1024 512 384 256; do
  timeout 300 python bench.py --config c0 --chunk $ch --steps 20 --warmup 3 --no-cpu --e2e-steps 1 --trace gpurun_out/tr_c0_$ch.json > gpurun_out/chunk_c0_$ch.log 2>&1; echo $ch rc=$?
done
for ch in 4096 2048 1024; do
  timeout 300 python bench.py --config c3 --chunk $ch --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/chunk_c3_$ch.log 2>&1; echo c3 $ch rc=$?
done

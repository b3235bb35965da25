# 2D chunk sweep (configs 0 and 1)
mkdir -p gpurun_out/ch
for c in c0 c1; do for ch in 8192 2048 1024 512 256; do
timeout 300 python bench.py --config $c --chunk $ch --steps 20 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ch/ab_${c}_ch${ch}_1.log 2>&1; echo $c $ch rc=$?
done; done

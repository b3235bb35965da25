# 3D chunk sweep (configs 2, 4s, 3)
mkdir -p gpurun_out/ch3
for c in c2 c4s c3; do for ch in 8192 12288 16384 32768; do
timeout 600 python bench.py --config $c --chunk $ch --steps 5 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/ch3/ab_${c}_ch${ch}_1.log 2>&1; echo $c $ch rc=$?
done; done

# where K1 time goes on the sparse background (config 4 slab) vs config 2: no run flushes (1), no Phase B (2)
mkdir -p gpurun_out/abl
for c in c4s c3; do for ab in 0 1 2; do
B200PIC_ABLATE=$ab timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/abl/${c}_$ab.log 2>&1; echo $c ab$ab rc=$?
done; done

for ab in 0 1 2 4 7; do
B200PIC_ABLATE=$ab timeout 600 python bench.py --config c2 --steps 3 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ablate_$ab.log 2>&1; echo ab$ab rc=$?
done

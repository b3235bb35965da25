# per-particle cost vs density: config 2 geometry at 2 / 4 / 8 / 16 particles per cell per species
mkdir -p gpurun_out/dens
for p in 2 4 8 16; do
timeout 600 python bench.py --config c2 --ppc $p --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/dens/c2_ppc$p.log 2>&1; echo ppc $p rc=$?
done

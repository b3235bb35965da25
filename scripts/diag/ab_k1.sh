# K1 A/B on config 2: default (interleaved, per-species rounding), without the low-bits updates, per-species items
B="python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 1"
timeout 300 $B > gpurun_out/ab_il.log 2>&1; echo rc=$?
B200PIC_ABLATE=16 timeout 300 $B > gpurun_out/ab_il_nolb.log 2>&1; echo rc=$?
timeout 300 $B --merge 0 > gpurun_out/ab_m0.log 2>&1; echo rc=$?

T=${T:-384}
B200PIC_K1_THREADS=$T python paper_2204_12837_b200/build_ext.py --force > gpurun_out/build_t.log 2>&1; echo build=$?
B200PIC_K1_THREADS=$T timeout 600 python bench.py --config c2 --steps 3 --warmup 1 --no-cpu --e2e-steps 1 --stage 0 > gpurun_out/t${T}.log 2>&1; echo t=$?
B200PIC_K1_THREADS=$T B200PIC_ABLATE=2 timeout 600 python bench.py --config c2 --steps 3 --warmup 1 --no-cpu --e2e-steps 1 --stage 0 > gpurun_out/t${T}_ab2.log 2>&1; echo tab2=$?

B200PIC_K1_THREADS=512 python paper_2204_12837_b200/build_ext.py --force > gpurun_out/build512.log 2>&1; echo build=$?
B200PIC_K1_THREADS=512 timeout 600 python bench.py --config c2 --steps 3 --warmup 1 --no-cpu --e2e-steps 1 --stage 0 > gpurun_out/t512.log 2>&1; echo t512=$?
B200PIC_K1_THREADS=512 B200PIC_ABLATE=2 timeout 600 python bench.py --config c2 --steps 3 --warmup 1 --no-cpu --e2e-steps 1 --stage 0 > gpurun_out/t512_ab2.log 2>&1; echo t512ab2=$?

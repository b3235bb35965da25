# A/B: z-pair consumer runs, cp.async staging; plus one ncu capture of the z-pair K1
bash scripts/gpu_ab.sh c2 2 zp1 zp0 zp0cp0
bash scripts/gpu_ab.sh c4s 1 zp1 zp0 zp0cp0
B="python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1"
B200PIC_LIB_PATH=$PWD/paper_2204_12837_b200/_build/exp/zp1.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 1 -o gpurun_out/k1_zp1 $B > gpurun_out/ncu_zp1.log 2>&1; echo ncu=$?

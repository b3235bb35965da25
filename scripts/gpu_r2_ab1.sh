# round 2: A/B of the per-species low-bits tile (WS_LB) and the TMA g8 staging on config 2, + K1 full capture
mkdir -p gpurun_out/ab1
B="python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 1"
for t in base lb0; do
  for g in 0 1; do
    e=""; [ $g = 1 ] && e="B200PIC_NO_G8=1"
    timeout 400 env $e B200PIC_LIB_PATH=$PWD/paper_2204_12837_b200/_build/exp/$t.so $B > gpurun_out/ab1/ab_${t}_nog8${g}_c2.log 2>&1; echo $t $g rc=$?
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_ -s 6 -c 1 -o gpurun_out/ab1/k1_c2 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ab1/ncu_full.log 2>&1; echo ncu=$?

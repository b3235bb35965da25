# ncu --set full of K1 for alternative builds: bash scripts/diag/prof_libs.sh tag...
E=$PWD/paper_2204_12837_b200/_build/exp
for t in "$@"; do
B="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --e2e-steps 1"
timeout 600 env B200PIC_LIB_PATH=$E/$t.so ncu --set full --clock-control none --import-source on -k regex:k1_ws -s 1 -c 1 -o gpurun_out/k1p_$t $B > gpurun_out/ncup_$t.log 2>&1; echo $t rc=$?
done

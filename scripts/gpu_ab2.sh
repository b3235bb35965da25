cfg=$1; ch=$2; shift 2
for t in "$@"; do
  timeout 300 env B200PIC_LIB_PATH=$PWD/paper_2204_12837_b200/_build/exp/$t.so python bench.py --config $cfg --chunk $ch --steps 5 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/ab2_${cfg}_${t}.log 2>&1; echo $t rc=$?
done

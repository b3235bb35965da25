# A/B across builds and chunk sizes: bash scripts/gpu_ab3.sh <config> "<tag:chunk> ..."
cfg=$1; shift
for tc in "$@"; do t=${tc%%:*}; ch=${tc#*:}
  timeout 300 env B200PIC_LIB_PATH=$PWD/paper_2204_12837_b200/_build/exp/$t.so python bench.py --config $cfg --chunk $ch --steps 5 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/ab3_${cfg}_${t}_${ch}.log 2>&1; echo $t $ch rc=$?
done

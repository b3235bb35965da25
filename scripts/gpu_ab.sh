# A/B of alternative builds (_build/exp/*.so), interleaved, repeated: bash scripts/gpu_ab.sh <config> <reps> tag...
cfg=$1; reps=$2; shift 2
for r in $(seq $reps); do for t in "$@"; do
  timeout 300 env B200PIC_LIB_PATH=$PWD/paper_2204_12837_b200/_build/exp/$t.so python bench.py --config $cfg --steps 5 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/ab_${cfg}_${t}_$r.log 2>&1; echo $t $r rc=$?
done; done

# interleaved A/B of (lib, env, args) variants, repeated: bash scripts/diag/ab_env.sh REPS "tag|lib|ENV=1 ENV2=2|args" ...
reps=$1; shift
E=$PWD/paper_2204_12837_b200/_build/exp
for r in $(seq $reps); do for spec in "$@"; do
  IFS='|' read -r tag lib envs args <<< "$spec"
  timeout 300 env B200PIC_LIB_PATH=$E/$lib.so $envs python bench.py --steps 8 --warmup 3 --no-cpu --e2e-steps 1 $args > gpurun_out/abx_${tag}_$r.log 2>&1; echo $tag $r rc=$?
done; done

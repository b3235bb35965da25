# A/B with an environment setting: bash scripts/gpu_ab_env.sh <config> "<ENV=V ...>" tag...
cfg=$1; envs=$2; shift 2
for t in "$@"; do
  timeout 300 env $envs B200PIC_LIB_PATH=$PWD/paper_2204_12837_b200/_build/exp/$t.so python bench.py --config $cfg --steps 5 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/abe_${cfg}_${t}.log 2>&1; echo $t rc=$?
done

# Parametrised A/B runner (replaces the per-experiment gpu_ab*.sh recipes):
#   CONFIGS="c2 c4s" REPS=1 ENVS="X=1" bash scripts/ab.sh OUTDIR tag1 tag2 ...
# each tag is an alternative build paper_2204_12837_b200/_build/exp/<tag>.so (scripts/build_exp.sh);
# summary: python scripts/ab_table.py OUTDIR/*.log
out=$1; shift
mkdir -p $out
for r in $(seq 1 ${REPS:-1}); do
  for c in ${CONFIGS:-c2}; do
    for t in "$@"; do
      timeout 400 env $ENVS B200PIC_LIB_PATH=$PWD/paper_2204_12837_b200/_build/exp/$t.so \
        python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu --e2e-steps 1 > $out/${c}-${t}_r$r.log 2>&1
      echo "$c $t rc=$?"
    done
  done
done

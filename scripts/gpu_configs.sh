# bench lines of the imbalanced configs (per-particle time vs config 2)
mkdir -p gpurun_out/cfg
for c in c3 c4s c1; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/cfg/bench_$c.log 2>&1; echo bench $c rc=$?
done

# one bench line per BASELINE config (single GPU): bash scripts/diag/all_configs.sh TAG
TAG=${1:-x}
for c in c2 c3 c4s c1 c0; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/cfg_${TAG}_$c.log 2>&1; echo $c rc=$?
done

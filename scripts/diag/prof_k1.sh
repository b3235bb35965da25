# ncu captures of K1 on config 2 for two item modes (usage: bash scripts/diag/prof_k1.sh TAG)
TAG=${1:-x}
for M in 2 0; do
B="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 --merge $M"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_ws -s 1 -c 1 -o gpurun_out/k1_${TAG}_m$M $B > gpurun_out/ncu_${TAG}_m$M.log 2>&1; echo ncu_m${M}_rc=$?
done

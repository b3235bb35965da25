# K1 ncu captures of the imbalanced 3D configs (3 and 4s)
mkdir -p gpurun_out/pi
for c in c4s c3; do
B="python bench.py --config $c --steps 2 --warmup 1 --no-cpu --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 1 -o gpurun_out/pi/k1_$c $B > gpurun_out/pi/ncu_$c.log 2>&1; echo ncu $c rc=$?
done

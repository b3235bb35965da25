# one full ncu capture of the warp-specialised K1 on config 2
B="python bench.py --variant 2 --steps 2 --warmup 1 --no-cpu --e2e-steps 1"
$B > gpurun_out/plain_ws.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_ws -s 2 -c 1 -o gpurun_out/k1_ws $B > gpurun_out/ncu_ws.log 2>&1; echo ncu=$?

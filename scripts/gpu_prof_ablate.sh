B="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 --stage 1"
export B200PIC_ABLATE=${AB:-7}
$B > gpurun_out/plain_ab.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fused -s 1 -c 1 -o gpurun_out/k1_ab$B200PIC_ABLATE $B > gpurun_out/ncu_ab.log 2>&1; echo ncu_rc=$?

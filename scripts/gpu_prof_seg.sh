B="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --e2e-steps 1"
$B > gpurun_out/plain_seg.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_seg_tiles -s 3 -c 1 -o gpurun_out/seg_c2 $B > gpurun_out/ncu_seg.log 2>&1; echo ncu_rc=$?

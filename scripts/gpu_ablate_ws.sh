for a in 0 1 2 4 8; do
  timeout 300 env B200PIC_ABLATE=$a python bench.py --config c2 --steps 3 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/abl_$a.log 2>&1; echo $a rc=$?
done

mkdir -p gpurun_out/tr4
for sch in on off; do
  timeout 600 python bench.py --config c4s --schedule $sch --steps 3 --warmup 2 --no-cpu --e2e-steps 1 \
    --trace gpurun_out/tr4/trace_c4s_${sch}.json > gpurun_out/tr4/trace_c4s_${sch}.log 2>&1; echo trace $sch rc=$?
  gzip -f gpurun_out/tr4/trace_c4s_${sch}.json
done

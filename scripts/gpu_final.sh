# round-end measurements: every config's bench line (with the CPU baseline), reference arm, traces
mkdir -p gpurun_out/final
for c in c2 c0 c1 c3 c4s; do
  timeout 900 python bench.py --config $c > gpurun_out/final/bench_$c.log 2>&1; echo bench $c rc=$?
done
timeout 900 python bench.py --impl reference > gpurun_out/final/ref_c2.log 2>&1; echo ref rc=$?
timeout 600 python bench.py --config c0 --graph > gpurun_out/final/bench_c0_graph.log 2>&1; echo graph rc=$?
for c in c3 c0; do for sch in on off; do
  timeout 600 python bench.py --config $c --schedule $sch --steps 5 --warmup 3 --no-cpu --e2e-steps 1 \
    --trace gpurun_out/final/trace_${c}_${sch}.json > gpurun_out/final/trace_${c}_${sch}.log 2>&1; echo trace $c $sch rc=$?
  gzip -f gpurun_out/final/trace_${c}_${sch}.json
done; done

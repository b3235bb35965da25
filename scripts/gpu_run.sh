# One parametrised recipe for every gpurun measurement (folds the round-1 one-off gpu_*.sh scripts).
#   bash scripts/gpu_run.sh MODE [args]   (run under /usr/local/graft/bin/gpurun; outputs in gpurun_out/)
# MODE
#   tests                     pytest -m gpu (+ smoke)                           -> gpurun_out/tests/
#   bench  "c2 c3 ..." [steps] bench lines without the CPU leg                 -> gpurun_out/bench/
#   launches CFG              ncu launch list (gpu__time_duration, cold cache)  -> gpurun_out/prof/launches_CFG.csv
#   capture CFG [skip]        ncu --set full of one K1 launch                   -> gpurun_out/prof/k1_CFG.ncu-rep
#   ab OUT "cfgs" tags...     alternative builds _build/exp/<tag>.so (scripts/build_exp.sh), same box (scripts/ab.sh)
#   density                   config-2 geometry at 2/4/8/16 ppc/species         -> gpurun_out/dens/
#   trace CFG                 K1 work-item traces, queue on and off             -> gpurun_out/trace/
#   final                     round-end: every config with its CPU baseline, the reference arm, the CUDA-graph
#                             line of config 0, traces of configs 3 and 0       -> gpurun_out/final/
mode=$1; shift
B="python bench.py --no-cpu --e2e-steps 1 --warmup 3"
case $mode in
tests)
  mkdir -p gpurun_out/tests
  timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/tests/gpu.log 2>&1; echo gpu_tests=$?
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/tests/smoke.log 2>&1; echo smoke=$? ;;
bench)
  mkdir -p gpurun_out/bench
  for c in ${1:-c2}; do timeout 600 $B --config $c --steps ${2:-10} > gpurun_out/bench/bench_$c.log 2>&1; echo $c=$?; done ;;
launches)
  mkdir -p gpurun_out/prof
  timeout 600 $B --config $1 --steps 2 > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/prof/launches_$1.csv $B --config $1 --steps 2 > gpurun_out/prof/ncu_launch_$1.log 2>&1
  echo launches=$? ;;
capture)
  mkdir -p gpurun_out/prof
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k1_ -s ${2:-6} -c 1 \
    -o gpurun_out/prof/k1_$1 $B --config $1 --steps 1 > gpurun_out/prof/ncu_full_$1.log 2>&1; echo capture=$? ;;
ab)
  out=$1; cfgs=$2; shift 2; CONFIGS="$cfgs" bash scripts/ab.sh $out "$@" ;;
density)
  mkdir -p gpurun_out/dens
  for p in 2 4 8 16; do timeout 600 $B --config c2 --ppc $p --steps 10 > gpurun_out/dens/c2_ppc$p.log 2>&1; echo ppc $p=$?; done ;;
trace)
  mkdir -p gpurun_out/trace
  for sch in on off; do
    timeout 600 $B --config $1 --schedule $sch --steps 3 --trace gpurun_out/trace/trace_$1_$sch.json \
      > gpurun_out/trace/trace_$1_$sch.log 2>&1; echo trace $sch=$?
    gzip -f gpurun_out/trace/trace_$1_$sch.json
  done ;;
final)
  mkdir -p gpurun_out/final
  for c in c2 c0 c1 c3 c4s; do timeout 900 python bench.py --config $c > gpurun_out/final/bench_$c.log 2>&1; echo bench $c=$?; done
  timeout 900 python bench.py --impl reference > gpurun_out/final/ref_c2.log 2>&1; echo ref=$?
  timeout 600 python bench.py --config c0 --graph > gpurun_out/final/bench_c0_graph.log 2>&1; echo graph=$?
  for c in c3 c0; do for sch in on off; do
    timeout 600 $B --config $c --schedule $sch --steps 5 --trace gpurun_out/final/trace_${c}_${sch}.json \
      > gpurun_out/final/trace_${c}_${sch}.log 2>&1; echo trace $c $sch=$?
    gzip -f gpurun_out/final/trace_${c}_${sch}.json
  done; done ;;
*) echo "unknown mode $mode"; exit 2 ;;
esac

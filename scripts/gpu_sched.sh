for c in c1 c3 c4s; do for sch in on off; do
timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu --e2e-steps 1 --schedule $sch > gpurun_out/sched_${c}_${sch}.log 2>&1; echo ${c}_${sch}=$?
done; done

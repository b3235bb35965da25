run() { timeout 300 env $2 python bench.py --config c2 --variant 2 --steps 5 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/wsr_$1.log 2>&1; echo $1 rc=$?; }
run base ""
for t in r176_80 r160_96 r184_72; do run $t B200PIC_LIB_PATH=$PWD/paper_2204_12837_b200/_build/exp/$t.so; done

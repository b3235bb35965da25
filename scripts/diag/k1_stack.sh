# Registers / stack of the benchmarked K1 instantiations (dense config 2, sparse config 4s) without a GPU:
#   bash scripts/diag/k1_stack.sh [-DNAME=V ...]
# A producer allocation flip shows up here as STACK growing past 24 / 48 bytes (round 2: one pitch constant
# took the dense kernel to 184 bytes and K1 from 62 to 73 ms).
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false --expt-relaxed-constexpr -cubin "$@" \
  -o /tmp/k1_stack.cubin paper_2204_12837_b200/csrc/k1_particles.cu 2>&1 | grep -i " error" && exit 1
cuobjdump -res-usage /tmp/k1_stack.cubin 2>/dev/null | \
  grep -A1 "k1_wsILi3ELb1ELi1ELb1ELb0ELb1ELb0E\|k1_wsILi3ELb1ELi1ELb1ELb1ELb1ELb0E" | grep -o "Function.*k1_wsILi3[^ ]*\|REG:[0-9]* STACK:[0-9]*"

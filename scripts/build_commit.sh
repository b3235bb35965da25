# build the CUDA library of an older commit into _build/exp/<tag>.so (A/B timing against the same box)
set -e
commit=$1; tag=$2; shift 2
d=$(mktemp -d)
git archive $commit paper_2204_12837_b200/csrc include | tar -x -C $d
mkdir -p paper_2204_12837_b200/_build/exp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr "$@" -o paper_2204_12837_b200/_build/exp/$tag.so $d/paper_2204_12837_b200/csrc/*.cu
rm -rf $d

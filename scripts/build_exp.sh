# alternative builds for tuning experiments: _build/exp/<tag>.so (load with B200PIC_LIB_PATH)
mkdir -p paper_2204_12837_b200/_build/exp
# (existing builds are kept; delete _build/exp to start over)
b() { B200PIC_EXTRA_DEFS="$2" B200PIC_BUILD_OUT=$PWD/paper_2204_12837_b200/_build/exp/$1.so python -c "from paper_2204_12837_b200 import build_ext; build_ext.build(force=True)" || echo FAIL $1; }
for spec in "$@"; do tag=${spec%%:*}; defs=${spec#*:}; b $tag "$defs" & done
wait

# alternative builds for tuning experiments: _build/exp/<tag>.so (load with B200PIC_LIB_PATH)
mkdir -p paper_2204_12837_b200/_build/exp
b() { B200PIC_EXTRA_DEFS="$2" B200PIC_BUILD_OUT=$PWD/paper_2204_12837_b200/_build/exp/$1.so python -c "from paper_2204_12837_b200 import build_ext; build_ext.build(force=True)" || echo FAIL $1; }
b r176_80 "-DWS_PREG=176 -DWS_CREG=80" &
b r160_96 "-DWS_PREG=160 -DWS_CREG=96" &
b r184_72 "-DWS_PREG=184 -DWS_CREG=72" &
wait

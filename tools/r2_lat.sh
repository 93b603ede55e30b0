# single-scan latency of library variants (VARIANTS="base nopdl")
for v in ${VARIANTS}; do lib=$PWD/paper_2005_02704_b200/liblidarseg_b200.so; [ "$v" != base ] && lib=$PWD/paper_2005_02704_b200/liblidarseg_b200_$v.so
LSEG_LIB_PATH=$lib timeout 300 python tools/latency.py $v 2>&1 | tail -1; done

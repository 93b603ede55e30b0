# full ncu capture of one kernel (KERNEL regex) for several library variants (LIBS="r1 base")
F=${FRAMES:-128}
for v in ${LIBS}; do
  lib=$PWD/paper_2005_02704_b200/liblidarseg_b200.so; [ "$v" != base ] && lib=$PWD/paper_2005_02704_b200/liblidarseg_b200_$v.so
  CMD="python tools/prof_run.py --frames $F --iters 2 --interval ${INTERVAL:-1}"
  LSEG_LIB_PATH=$lib $CMD > gpurun_out/prof_plain_$v.log 2>&1 || { echo "plain run $v failed"; continue; }
  LSEG_LIB_PATH=$lib timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^${KERNEL}\$" -s 1 -c 1 \
    -o gpurun_out/prof_${KERNEL}_$v $CMD > gpurun_out/ncu_${KERNEL}_$v.log 2>&1; echo "$v rc=$?"
done

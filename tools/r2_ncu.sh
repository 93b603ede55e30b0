# full ncu capture of named kernels (regex) on the prof_run driver: KERNELS="k_tile2 ..." FRAMES=128
F=${FRAMES:-128}
CMD="python tools/prof_run.py --frames $F --iters 2 --interval ${INTERVAL:-1}"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/prof_plain.log; exit 1; }
for k in ${KERNELS}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^$k\$" -s 1 -c 1 -o gpurun_out/prof_$k${TAG:-} $CMD \
    > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done

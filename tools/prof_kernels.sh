# full ncu capture of each named kernel (one launch each) on the 128-frame driver
# usage: bash tools/prof_kernels.sh k_tile_cc k_labels_backfill ...
CMD="python tools/prof_run.py --frames ${FRAMES:-128} --iters 2 --interval ${INTERVAL:-1}"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k "regex:^$k\$" -s 1 -c 1 -o gpurun_out/prof_$k $CMD \
    > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done

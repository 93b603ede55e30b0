# round-2 evidence: default bench line, ncu launch lists (time + DRAM bytes) at k = 1 and 5,
# one full ncu capture of k_tile (all on the 512-frame bench batch via tools/prof_run.py)
mkdir -p gpurun_out/ev
timeout 900 python bench.py > gpurun_out/ev/bench_default.json 2> gpurun_out/ev/bench_default.err; echo bench rc=$?
for k in 1 5; do
  CMD="python tools/prof_run.py --frames 512 --iters 2 --interval $k"
  $CMD > gpurun_out/ev/plain_k$k.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k 'regex:^k_' --csv --log-file gpurun_out/ev/launches_k$k.csv $CMD > gpurun_out/ev/ncu_launch_k$k.log 2>&1; echo launches k$k rc=$?
done
CMD="python tools/prof_run.py --frames 512 --iters 2 --interval 1"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_tile$' -s 1 -c 1 -o gpurun_out/ev/full_k_tile $CMD \
  > gpurun_out/ev/ncu_full.log 2>&1; echo full rc=$?

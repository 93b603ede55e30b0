# round-2 baseline: GPU tests, short bench, ncu launch list with DRAM bytes for every pipeline kernel
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-latency > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err; echo bench rc=$?
CMD="python tools/prof_run.py --frames 512 --iters 2 --interval ${INTERVAL:-1}"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k 'regex:^k_' --csv --log-file gpurun_out/launches_dram.csv $CMD > gpurun_out/ncu1.log 2>&1; echo ncu rc=$?

# the default bench line (timed)
start=$(date +%s)
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_def.json 2> gpurun_out/bench_def.err; echo bench rc=$? secs=$(( $(date +%s) - start ))
tail -3 gpurun_out/bench_def.err

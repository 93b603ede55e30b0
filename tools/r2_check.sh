# GPU tests + the default bench line
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/gputest.log
/usr/bin/time -v timeout 900 python bench.py > gpurun_out/bench_def.json 2> gpurun_out/bench_def.err; echo bench rc=$?
tail -3 gpurun_out/bench_def.err

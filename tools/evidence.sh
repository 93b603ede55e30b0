# round evidence: full bench line, then the ncu launch list and one full capture of the top kernel
set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-latency --also-interval 0"
KRE='regex:^k_'
$CMD > gpurun_out/plain_ev.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --csv --log-file gpurun_out/launches_ev.csv $CMD > gpurun_out/ncu_ev1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:^k_tile$" -s 3 -c 1 -o gpurun_out/prof_ev $CMD > gpurun_out/ncu_ev2.log 2>&1; echo ncu rc=$?

# quick: GPU parity tests (fast subset) + short bench with stage times
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:-} > gpurun_out/gputest.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gputest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-latency --no-accuracy --no-parity --also-intervals 5 ${BENCH_ARGS:-} > gpurun_out/bq.json 2> gpurun_out/bq.err; echo bench rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bq.json').read().strip().splitlines()[-1])
print("ms/step", round(d['ms_per_step'],4), "k5", round(d['other_intervals'][0]['ms_per_step'],4) if d['other_intervals'] else None)
print({k:v['ms'] for k,v in d['stages'].items()})
PY

# quick GPU check: parity tests + a 128-frame bench with stage times
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --frames ${FRAMES:-128} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-latency 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stage_ms'])"

# frame chunks on concurrent streams (--streams) and sequential chunks (--chunk) vs one launch
Q="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-latency --no-accuracy --no-parity --also-intervals ''"
for n in 1 2 4 8; do eval python bench.py --streams $n $Q 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('streams', $n, round(d['ms_per_step'],4), round(d['value']/1e9,3))"; done
for c in 0 16 32 64 128; do eval python bench.py --chunk $c $Q 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk', $c, round(d['ms_per_step'],4), round(d['value']/1e9,3), {k: v['ms'] for k, v in d['stages'].items()})"; done

# time library variants built by _build.build(defines=..., out=...): bash tools/variants.sh a b c
for v in "" "$@"; do lib=$PWD/paper_2005_02704_b200/liblidarseg_b200${v:+_$v}.so
LSEG_LIB_PATH=$lib timeout 300 python bench.py --frames ${FRAMES:-128} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-latency ${BENCH_ARGS:-} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), d['stage_ms'])"; done

# time library variants in the given order, each twice: bash tools/variants2.sh base a b
# (variant v = paper_2005_02704_b200/liblidarseg_b200_$v.so built with _build.build(defines=..., out=...))
for v in "$@"; do lib=$PWD/paper_2005_02704_b200/liblidarseg_b200.so; [ "$v" != base ] && lib=$PWD/paper_2005_02704_b200/liblidarseg_b200_$v.so
for rep in 1 2; do
LSEG_LIB_PATH=$lib timeout 300 python bench.py --frames ${FRAMES:-512} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-latency --no-accuracy --no-parity --also-intervals "${ALSO:-}" ${BENCH_ARGS:-} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $rep, round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['stages'].items()}, [round(o['ms_per_step'],4) for o in d['other_intervals']])"; done; done

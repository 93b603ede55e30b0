# time library variants in the given order, each twice (first run discarded): bash tools/variants2.sh base a b
for v in "$@"; do lib=$PWD/paper_2005_02704_b200/liblidarseg_b200.so; [ "$v" != base ] && lib=$PWD/paper_2005_02704_b200/liblidarseg_b200_$v.so
for rep in 1 2; do
LSEG_LIB_PATH=$lib timeout 300 python bench.py --frames ${FRAMES:-128} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-latency --also-interval 0 ${BENCH_ARGS:-} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $rep, round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms'].items()})"; done; done

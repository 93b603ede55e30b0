# throughput of each BASELINE config shape (device-resident batches), k = 1 and 5
for c in "vlp16 512" "hdl64_batch 512" "os128 256" "stress 64"; do set -- $c
python bench.py --config $1 --frames $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-latency --no-accuracy --no-parity --also-intervals 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); o=(d.get('other_intervals') or [{}])[0]
print('$1', '$2', 'k1: %.3f ms/step %.2f Gpts/s %.0f fr/s frac %.3f' % (d['ms_per_step'], d['value']/1e9, d['frames_per_s'], d['pipeline_roofline']['frac']), '| k5: %.3f ms %.2f Gpts/s frac %.3f' % (o.get('ms_per_step',0), o.get('value',0)/1e9, o.get('pipeline_frac',0)), {k: v['ms'] for k, v in d['stages'].items()})"
done

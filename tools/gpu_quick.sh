# quick perf check: bench several configs (+ optional mix override) without tests
TAG=${1:-q}; shift
for c in "$@"; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --sustain-seconds 0.3 > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
  python -c "
import json
d=json.load(open('gpurun_out/bench_${c}_$TAG.json')); r=d['roofline']
print('$c', d['config']['workload'].split(':')[0], 'value %.3e'%d['value'], 'kern %.3e frac %.3f'%(r['achieved'], r['frac']), d['config']['strategy'], 'cold', d['config'].get('cold_rerun_chunks_last_step'))
" || tail -5 gpurun_out/bench_${c}_$TAG.err
done

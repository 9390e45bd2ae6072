# paired (NEXT-2) tests + bench lines per mix
timeout 600 python -m pytest tests -m gpu -x -q -k "paired" 2>&1 | tail -4
for mix in full paper ieee; do
timeout 300 python bench.py --config n2 --mix $mix --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --sustain-seconds 0.3 > gpurun_out/bench_n2_$mix.json 2> gpurun_out/bench_n2.err
python -c "
import json; d=json.load(open('gpurun_out/bench_n2_$mix.json')); r=d['roofline']
print('n2 $mix value %.3e'%d['value'], 'ms %.3f'%d['ms_per_step'], 'GB/s %.0f frac %.3f'%(r['achieved'], r['frac']), 'alu frac %.4f'%r['alu_view']['frac'])
" || tail -5 gpurun_out/bench_n2.err
done

# usage: bash tools/sweep_tune.sh TAG "cfg:tune cfg:tune ..."   (tune "-" = defaults)
TAG=$1; shift
for ct in $@; do
  c=${ct%%:*}; t=${ct#*:}
  a=""; [ "$t" != "-" ] && a="--tune $t"
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --sustain-seconds 0.3 $a > gpurun_out/sw_$TAG.json 2> gpurun_out/sw_$TAG.err
  python -c "
import json
d=json.load(open('gpurun_out/sw_$TAG.json')); r=d['roofline']
print('$c $t', 'value %.3e'%d['value'], 'kern %.3e frac %.3f'%(r['achieved'], r['frac']), 'cold', d['config'].get('cold_rerun_chunks_last_step'))
" || tail -3 gpurun_out/sw_$TAG.err
done

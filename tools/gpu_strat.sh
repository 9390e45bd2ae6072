# usage: bash tools/gpu_strat.sh TAG CONFIG strategy...   (quick bench lines with a forced strategy)
TAG=$1; C=$2; shift 2
mkdir -p gpurun_out
for st in "$@"; do
  timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --sustain-seconds 0.3 --strategy $st > gpurun_out/strat_${C}_${TAG}_$st.json 2> gpurun_out/strat_${C}_${TAG}_$st.err
  python -c "
import json
d=json.load(open('gpurun_out/strat_${C}_${TAG}_$st.json')); r=d['roofline']
print('$C', '$st', 'value %.3e'%d['value'], 'kern %.3e frac %.3f'%(r['achieved'], r['frac']), 'ms %.3f'%d['ms_per_step'])
" || tail -3 gpurun_out/strat_${C}_${TAG}_$st.err
done

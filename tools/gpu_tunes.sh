# usage: bash tools/gpu_tunes.sh TAG CONFIG "tune1" "tune2" ...   ("-" = defaults)
TAG=$1; C=$2; shift 2
mkdir -p gpurun_out
i=0
for t in "$@"; do
  i=$((i+1))
  if [ "$t" = "-" ]; then TA=""; else TA="--tune $t"; fi
  timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --sustain-seconds 0.3 $TA > gpurun_out/tune_${C}_${TAG}_$i.json 2> gpurun_out/tune_${C}_${TAG}_$i.err
  python -c "
import json
d=json.load(open('gpurun_out/tune_${C}_${TAG}_$i.json')); r=d['roofline']
print('$C', '$t', 'value %.3e'%d['value'], 'kern %.3e frac %.3f'%(r['achieved'], r['frac']), 'ms %.3f'%d['ms_per_step'], 'cold', d['config'].get('cold_rerun_chunks_last_step'))
" || tail -3 gpurun_out/tune_${C}_${TAG}_$i.err
done

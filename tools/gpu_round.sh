# usage: bash tools/gpu_round.sh TAG [configs...]   (run on the GPU box via gpurun)
TAG=${1:-x}; shift
CONFIGS=${@:-c2 c3 c4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -x 2>&1 | tail -15 > gpurun_out/gpu_tests_$TAG.log
cat gpurun_out/gpu_tests_$TAG.log
for c in $CONFIGS; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/bench_${c}_$TAG.json')); r=d['roofline']
print('$c', 'value %.3e'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'kern %.3e frac %.3f'%(r['achieved'], r['frac']), d['config']['strategy'], 'e2e %.3e'%d['e2e']['value'], d['clocks'])
" || tail -5 gpurun_out/bench_${c}_$TAG.err
done
if [ -n "$NCU" ]; then
  for c in $NCU; do
    k=inter; [ "$c" = "c3" ] && k=intra
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_$k -s 2 -c 1 -o gpurun_out/prof_${c}_$TAG python bench.py --config $c --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --sustain-seconds 0 > gpurun_out/ncu_${c}_$TAG.log 2>&1
    tail -2 gpurun_out/ncu_${c}_$TAG.log
  done
fi

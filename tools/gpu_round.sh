# usage: bash tools/gpu_round.sh TAG [configs...]   (run on the GPU box via gpurun)
# GPU tests (all, no -x), then one bench line per config.
TAG=${1:-x}; shift
CONFIGS=${@:-c3 c2 c4 c5 c1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -rf --timeout 900 ${PYTEST_ARGS} -s 2>&1 > gpurun_out/gpu_tests_$TAG.full.log
tail -40 gpurun_out/gpu_tests_$TAG.full.log > gpurun_out/gpu_tests_$TAG.log
cat gpurun_out/gpu_tests_$TAG.log | tail -25
for c in $CONFIGS; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/bench_${c}_$TAG.json')); r=d['roofline']
print('$c', 'value %.3e'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'kern %.3e frac %.3f'%(r['achieved'], r['frac']), d['config']['strategy'], 'e2e %.3e'%(d['e2e'] or {}).get('value',0), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), d.get('graph_replay',{}).get('value'))
" || tail -5 gpurun_out/bench_${c}_$TAG.err
done

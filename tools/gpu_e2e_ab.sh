# pipelined e2e (EVOGP_E2E_DEPTH=2, default) vs one step at a time (=1), plus the streaming GPU tests
timeout 600 python -m pytest tests/test_gpu_tensorize.py -m gpu -q -k "streaming" 2>&1 | tail -2
for c in ${@:-c2 c3 c4}; do
  for dep in 1 2; do
    EVOGP_E2E_DEPTH=$dep timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --sustain-seconds 0 > /tmp/e.json 2>/tmp/e.err
    python -c "
import json; d=json.load(open('/tmp/e.json'))
print('$c depth $dep value %.3e e2e %.3e'%(d['value'], d['e2e']['value']), d['e2e']['path'])" || tail -3 /tmp/e.err
  done
done

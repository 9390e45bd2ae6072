# A/B an env knob on the full step value (kernel + compile pass): bash tools/gpu_value_ab.sh "A=1 A=2" configs...
SETTINGS=$1; shift
for st in $SETTINGS; do
  for c in "$@"; do
    env $st timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --sustain-seconds 0 > /tmp/b.json 2>/tmp/b.err
    python -c "
import json; d=json.load(open('/tmp/b.json')); r=d['roofline']
print('$st $c value %.3e kern %.3e frac %.3f ms %.3f' % (d['value'], r['achieved'], r['frac'], d['ms_per_step']))" 2>/dev/null || (echo "$st $c failed"; tail -3 /tmp/b.err)
  done
done

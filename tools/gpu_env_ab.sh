# A/B an environment knob: bash tools/gpu_env_ab.sh "VAR=a VAR=b" configs...
SETTINGS=$1; shift
for st in $SETTINGS; do
  for c in "$@"; do
    env $st timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --sustain-seconds 0 > /tmp/b.json 2>/tmp/b.err
    python -c "
import json; d=json.load(open('/tmp/b.json')); r=d['roofline']
print('$st $c kern %.3e frac %.3f cold %s' % (r['achieved'], r['frac'], d['config']['cold_rerun_chunks_last_step']))" 2>/dev/null || (echo "$st $c failed"; tail -3 /tmp/b.err)
  done
done

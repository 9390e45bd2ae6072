# env-knob A/B on several configs: bash tools/gpu_env_ab2.sh "ENV=VAL ..." configs...
ENVS=$1; shift
for c in $@; do
  st=20; wu=5; [ "$c" = "g1" ] && st=60 && wu=3
  env $ENVS timeout 300 python bench.py --config $c --steps $st --warmup $wu --no-cpu-baseline --no-e2e --sustain-seconds 0.3 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$ENVS] $c', '%.3e' % d['value'], 'kern %.3e frac %.3f' % (r['achieved'], r['frac']))"
done

# quick A/B numbers: GPU tests + device-timed value / kernel frac for a few configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -rf --timeout 600 2>&1 | tail -2
for c in ${@:-c2 c4 c5}; do
  st=20; wu=5; [ "$c" = "g1" ] && st=60 && wu=3
  timeout 300 python bench.py --config $c --steps $st --warmup $wu --no-cpu-baseline --no-e2e --sustain-seconds 0.5 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', '%.3e' % d['value'], 'kern %.3e frac %.3f' % (r['achieved'], r['frac']))"
done

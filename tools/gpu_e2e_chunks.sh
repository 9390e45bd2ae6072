# e2e chunk-count sweep at depth 2
for c in c2 c4; do for ch in 1 2 4 8; do
  EVOGP_E2E_CHUNKS=$ch timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --sustain-seconds 0 > /tmp/e.json 2>/tmp/e.err
  python -c "
import json; d=json.load(open('/tmp/e.json'))
print('$c chunks $ch e2e %.3e'%d['e2e']['value'])" || tail -3 /tmp/e.err
done; done

# e2e repeatability: default bench line flags, depth 2 / 1, twice
nproc; cat /proc/loadavg
for rep in 1 2; do for dep in 2 1; do
  EVOGP_E2E_DEPTH=$dep timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > /tmp/e.json 2>/tmp/e.err
  python -c "
import json; d=json.load(open('/tmp/e.json'))
print('c2 rep $rep depth $dep value %.3e e2e %.3e'%(d['value'], d['e2e']['value']))" || tail -3 /tmp/e.err
done; done
EVOGP_E2E_DEPTH=2 timeout 300 python bench.py --config c2 --steps 100 --warmup 5 --no-cpu-baseline > /tmp/e.json 2>/tmp/e.err
python -c "
import json; d=json.load(open('/tmp/e.json'))
print('c2 100 steps depth 2 value %.3e e2e %.3e'%(d['value'], d['e2e']['value']))"

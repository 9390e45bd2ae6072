for c in c2 c4 c3; do
  for w in 20 24 28 32; do
    EVOGP_TUNE_K=8 EVOGP_TUNE_WARPS=$w timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --sustain-seconds 0 > /tmp/b.json 2>/dev/null
    python -c "
import json; d=json.load(open('/tmp/b.json')); r=d['roofline']
print('$c K=8 W=$w kern %.3e frac %.3f cold %s' % (r['achieved'], r['frac'], d['config']['cold_rerun_chunks_last_step']))" 2>/dev/null || echo "$c W=$w failed"
  done
done

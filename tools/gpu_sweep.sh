# occupancy / K sweep on c2, c3, c4 (EVOGP_TUNE_K, EVOGP_TUNE_WARPS)
for c in c2 c4 c3; do
  for k in 4 8; do
    for w in 16 20 24 32 40; do
      EVOGP_TUNE_K=$k EVOGP_TUNE_WARPS=$w timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --sustain-seconds 0 > /tmp/b.json 2>/dev/null
      python -c "
import json; d=json.load(open('/tmp/b.json')); r=d['roofline']
print('$c K=$k W=$w kern %.3e frac %.3f cold %s' % (r['achieved'], r['frac'], d['config']['cold_rerun_chunks_last_step']))" 2>/dev/null || echo "$c K=$k W=$w failed"
    done
  done
done

# A/B the variant libraries in variants/*/ on the given configs (restores the in-tree build afterwards)
cp paper_2501_17168_b200/libevogp.so /tmp/libevogp.base.so
for v in base $(ls variants); do
  if [ "$v" = base ]; then cp /tmp/libevogp.base.so paper_2501_17168_b200/libevogp.so; else cp variants/$v/libevogp.so paper_2501_17168_b200/libevogp.so; fi
  for c in "$@"; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --sustain-seconds 0 > /tmp/b.json 2>/dev/null
    python -c "
import json; d=json.load(open('/tmp/b.json')); r=d['roofline']
print('$v $c kern %.3e frac %.3f cold %s' % (r['achieved'], r['frac'], d['config']['cold_rerun_chunks_last_step']))" 2>/dev/null || echo "$v $c failed"
  done
done
cp /tmp/libevogp.base.so paper_2501_17168_b200/libevogp.so

# A/B of k_paired: in-tree build (base) vs variants/$1 on n2, then the paired GPU tests on the variant
VS=${@:-split}
cp paper_2501_17168_b200/libevogp.so /tmp/libevogp.base.so
for v in base $VS; do
  [ "$v" = base ] || cp variants/$v/libevogp.so paper_2501_17168_b200/libevogp.so
  for mix in full paper; do
    timeout 300 python bench.py --config n2 --mix $mix --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --sustain-seconds 0.3 > /tmp/n2.json 2>/tmp/n2.err
    python -c "
import json; d=json.load(open('/tmp/n2.json')); r=d['roofline']
print('$v n2 $mix value %.3e'%d['value'], 'ms %.3f'%d['ms_per_step'], 'GB/s %.0f frac %.3f'%(r['achieved'], r['frac']))
" || tail -5 /tmp/n2.err
  done
done
for v in $VS; do cp variants/$v/libevogp.so paper_2501_17168_b200/libevogp.so; echo $v; timeout 600 python -m pytest tests -m gpu -x -q -k "paired" 2>&1 | tail -1; done
cp /tmp/libevogp.base.so paper_2501_17168_b200/libevogp.so

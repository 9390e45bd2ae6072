# A/B of the shared-stack budget (EVOGP_TUNE_WARPS = resident-warp target that sizes SD)
for w in 32 40 48 64; do
  for c in ${@:-c2 c4}; do
    st=20; wu=5; [ "$c" = "g1" ] && st=40 && wu=3
    EVOGP_TUNE_WARPS=$w timeout 300 python bench.py --config $c --steps $st --warmup $wu --no-cpu-baseline --no-e2e --sustain-seconds 0.3 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('warps=$w $c', '%.3e' % d['value'], 'kern %.3e frac %.3f' % (r['achieved'], r['frac']))"
  done
done

for c in "200 63 17 6 4096" "64 31 4 2 1000" "33 127 8 3 20001"; do for st in inter intra; do for m in eval cls; do
 echo "== $c $st $m"; timeout 40 python tools/dbg_cls.py $c $st $m 2>&1 | tail -3; echo "rc=$?"
done; done; done

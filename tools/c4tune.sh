for t in "" "reorder_above=12" "reorder_above=100"; do
  BENCH_ARGS="--tune $t" 
  [ -z "$t" ] && BENCH_ARGS=""
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$t.csv python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --sustain-seconds 0 $BENCH_ARGS > /dev/null 2>&1
  echo "tune=$t"; grep -E "k_prepare|k_inter" gpurun_out/l_$t.csv | awk -F'","' '{print $5, $NF}' | tail -2
done

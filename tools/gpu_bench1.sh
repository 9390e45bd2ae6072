set -x
mkdir -p gpurun_out
for c in c2 c1 c4 c3 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -3 gpurun_out/bench_$c.err
  cat gpurun_out/bench_$c.json
done
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_c2.json 2>&1; cat gpurun_out/bench_ref_c2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --sustain-seconds 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter -s 2 -c 1 -o gpurun_out/prof_c2_inter python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --sustain-seconds 0 > gpurun_out/ncu_c2.log 2>&1
tail -3 gpurun_out/ncu_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_intra -s 2 -c 1 -o gpurun_out/prof_c3_intra python bench.py --config c3 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --sustain-seconds 0 > gpurun_out/ncu_c3.log 2>&1
tail -3 gpurun_out/ncu_c3.log
ls -la gpurun_out

# ncu evidence for the NEXT-3/4 loop (bench g1): launch list + full captures of
# the three per-generation kernels after 20 warm-up generations
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_g1_$TAG.csv \
  python bench.py --config g1 --steps 5 --warmup 20 --no-cpu-baseline --no-e2e --sustain-seconds 0 > /dev/null 2>&1
for k in k_reproduce k_prepare k_eval; do
  rk=$k; [ $k = k_eval ] && rk="k_in(ter|tra)"  # the fitness kernel the selector picks
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rk" -s 22 -c 1 -o gpurun_out/prof_g1_${k}_$TAG \
    python bench.py --config g1 --steps 3 --warmup 20 --no-cpu-baseline --no-e2e --sustain-seconds 0 > gpurun_out/ncu_g1_${k}_$TAG.log 2>&1
  tail -1 gpurun_out/ncu_g1_${k}_$TAG.log
done
ls gpurun_out | grep $TAG

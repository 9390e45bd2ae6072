# usage: bash tools/gpu_prof_kern.sh TAG cfg kernel_regex  — ncu --set full capture of one kernel of a config
TAG=$1; c=$2; k=$3
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_${c}_${k}_$TAG \
  python bench.py --config $c --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --sustain-seconds 0 ${BENCH_ARGS} > gpurun_out/ncu_${c}_${k}_$TAG.log 2>&1
tail -1 gpurun_out/ncu_${c}_${k}_$TAG.log
ncu -i gpurun_out/prof_${c}_${k}_$TAG.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/sass_${c}_${k}_$TAG.csv.gz

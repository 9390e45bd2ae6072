# usage: bash tools/gpu_prof_src.sh TAG cfg...  — one ncu --set full capture of each config's dominant
# kernel (source-level SASS counts exported to CSV) for instruction-mix work
TAG=${1:-p}; shift
mkdir -p gpurun_out
kern() { case $1 in c3|c5) echo k_intra;; n2) echo k_paired;; *) echo k_inter;; esac; }
for c in "$@"; do
  k=$(kern $c)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_${c}_$TAG \
    python bench.py --config $c --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --sustain-seconds 0 ${BENCH_ARGS} > gpurun_out/ncu_${c}_$TAG.log 2>&1
  tail -1 gpurun_out/ncu_${c}_$TAG.log
  ncu -i gpurun_out/prof_${c}_$TAG.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/sass_${c}_$TAG.csv.gz
done

# usage: bash tools/gpu_profile.sh TAG [configs]  — ncu launch lists + full captures of the dominant kernels
TAG=${1:-r01}; shift
CONFIGS=${@:-c2 c3 c4 c5 c5b n2}
mkdir -p gpurun_out
kern() { case $1 in n2) echo k_paired;; *) echo "k_in(ter|tra)";; esac; }  # the eval kernel the selector picks
for c in $CONFIGS; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${c}_$TAG.csv \
    python bench.py --config $c --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --sustain-seconds 0 > /dev/null 2>&1
done
for c in $CONFIGS; do
  k=$(kern $c)
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 -o gpurun_out/prof_${c}_$TAG \
    python bench.py --config $c --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --sustain-seconds 0 > gpurun_out/ncu_${c}_$TAG.log 2>&1
  tail -1 gpurun_out/ncu_${c}_$TAG.log
done
ls gpurun_out | grep $TAG

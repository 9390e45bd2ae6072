# ncu --set full capture of the dominant eval kernel of one config: bash tools/gpu_prof_one.sh TAG CONFIG [bench args]
TAG=$1; C=$2; shift 2
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_in(ter|tra)" -s 2 -c 1 -o gpurun_out/prof1_${C}_$TAG \
  python bench.py --config $C --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --sustain-seconds 0 "$@" > gpurun_out/ncu1_${C}_$TAG.log 2>&1
tail -1 gpurun_out/ncu1_${C}_$TAG.log
python tools/ncu_summary.py gpurun_out/prof1_${C}_$TAG.ncu-rep --out gpurun_out/prof1_${C}_$TAG.json > /dev/null 2>&1
ncu -i gpurun_out/prof1_${C}_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/prof1_${C}_$TAG.sass.csv 2>/dev/null
gzip -f gpurun_out/prof1_${C}_$TAG.sass.csv
rm -f gpurun_out/prof1_${C}_$TAG.ncu-rep

# full refresh on the box: results, ncu launch lists + full captures, summaries;
# the .ncu-rep files are summarised there and removed (gpurun copies back <= 64 MiB)
TAG=${1:-r01}
bash tools/gpu_results.sh $TAG
bash tools/gpu_profile.sh $TAG
bash tools/gpu_profile_g1.sh $TAG
mkdir -p gpurun_out/summaries_$TAG
for r in gpurun_out/prof_*_$TAG.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py $r --out gpurun_out/summaries_$TAG/$b.json > /dev/null 2>&1 || echo "summary failed $b"
  ncu -i $r --page source --csv --print-source sass > gpurun_out/summaries_$TAG/$b.sass.csv 2>/dev/null
  gzip -f gpurun_out/summaries_$TAG/$b.sass.csv
done
rm -f gpurun_out/prof_*_$TAG.ncu-rep
du -sh gpurun_out

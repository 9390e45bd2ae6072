# usage: bash tools/sanitize.sh TAG   — compute-sanitizer (memcheck, racecheck, synccheck, initcheck)
# over tools/sanitize_run.py (every kernel of libevogp.so on small inputs); logs in gpurun_out/
TAG=${1:-s}
mkdir -p gpurun_out
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --target-processes all \
    python tools/sanitize_run.py > gpurun_out/sanitizer_${tool}_$TAG.log 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run ok' gpurun_out/sanitizer_${tool}_$TAG.log | tr '\n' ' ')"
done

# usage: bash tools/gpu_cycle.sh TAG "pytest selection" configs...  (on the GPU box via gpurun)
# GPU tests (selection), then a quick bench line per config
TAG=$1; SEL=$2; shift 2
mkdir -p gpurun_out
timeout 1500 python -m pytest $SEL -m gpu -q -x -rf --timeout 900 > gpurun_out/gpu_tests_$TAG.log 2>&1
tail -15 gpurun_out/gpu_tests_$TAG.log
bash tools/gpu_quick.sh $TAG "$@"

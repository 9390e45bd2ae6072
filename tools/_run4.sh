./tools/microbench/fastmath_tp | tee gpurun_out/fastmath_tp2.jsonl
python -m pytest tests/test_gpu_accuracy.py -q -x -s 2>&1 | grep -E "worst|passed|failed|Error|assert" | head -20
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in c5b c5 c3; do bash tools/gpu_tunes.sh $1 $c -; done

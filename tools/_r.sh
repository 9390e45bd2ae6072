python -m pytest tests -m gpu -q -x 2>&1 | tail -2
bash tools/gpu_tunes.sh fd c4 - fused_compile=1

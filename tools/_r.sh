bash tools/gpu_tunes.sh k16 c3 - K=16 K=16,target_warps=16 K=16,target_warps=24

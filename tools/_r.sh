bash tools/gpu_tunes.sh uc2 c2 - unit_chunks=2 unit_chunks=4

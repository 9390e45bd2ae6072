bash tools/gpu_prof_one.sh now c5

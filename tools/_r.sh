python -m pytest tests -m gpu -q -x -k "paired" 2>&1 | tail -2
timeout 600 python bench.py --config n2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/n2new.json 2> gpurun_out/n2new.err; python -c "
import json; d=json.load(open('gpurun_out/n2new.json')); r=d['roofline']; print('n2', d['value'], r['achieved'], r['unit'], r['frac'], d['ms_per_step'])"

# A/B of the compile-pass / stack knobs on the whole-run loop (bench g1)
mkdir -p gpurun_out
run() { echo "== $1"; env $2 timeout 300 python bench.py --config g1 --steps 60 --warmup 3 --no-cpu-baseline --no-e2e --sustain-seconds 0.3 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('value %.3e ms/gen %.2f kern %.3e share %s mean_len %.1f' % (d['value'], d['ms_per_step'], r['achieved'], r['step_share'], d['config']['mean_len']))"; }
run default ""
run above2 "EVOGP_TUNE_REORDER_ABOVE=2"
run above4 "EVOGP_TUNE_REORDER_ABOVE=4"
run above8 "EVOGP_TUNE_REORDER_ABOVE=8"
run k4 "EVOGP_TUNE_K=4"
run k4above2 "EVOGP_TUNE_K=4 EVOGP_TUNE_REORDER_ABOVE=2"
run k4above4 "EVOGP_TUNE_K=4 EVOGP_TUNE_REORDER_ABOVE=4"
run noreorder "EVOGP_TUNE_REORDER=0"

# usage: bash tools/gpu_results.sh TAG — one full bench line per config (with e2e and cpu_baseline)
TAG=${1:-r01}
mkdir -p gpurun_out/results_$TAG
for c in c1 c2 c3 c4 c5 c5b n2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/results_$TAG/$c.json 2> gpurun_out/results_$TAG/$c.err
done
timeout 600 python bench.py --config g1 --steps 100 --warmup 3 > gpurun_out/results_$TAG/g1.json 2> gpurun_out/results_$TAG/g1.err
python - <<PY
import json, glob, os
for f in sorted(glob.glob("gpurun_out/results_$TAG/*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(os.path.basename(f), "FAILED", e); continue
    r = d["roofline"]; e2e = d.get("e2e") or {}; cb = d.get("cpu_baseline") or {}
    print(os.path.basename(f), "value %.3e" % d["value"], "ms/step %.3f" % d["ms_per_step"],
          "kern %.3e %s frac %.3f" % (r["achieved"], r["unit"], r["frac"]), "e2e %.3e" % e2e.get("value", 0),
          "cpu %.3e" % cb.get("value", 0), d["clocks"].get("reasons"))
PY

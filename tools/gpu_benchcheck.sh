# the default bench line (cached measured selection) and the band projections, with K runs per CUDA graph
tag=${1:-r2p}
mkdir -p gpurun_out/$tag
( time timeout 1200 python bench.py ) > gpurun_out/$tag/bench.json 2> gpurun_out/$tag/bench.err
tail -3 gpurun_out/$tag/bench.err
python - <<PY
import json
d = json.loads(open("gpurun_out/$tag/bench.json").read().strip().splitlines()[-1])
print("headline", round(d["ms_per_step"] * 1e3, 2), "us", round(d["roofline"]["hbm"]["frac"], 3), d["config"]["launch"][:60], d["clocks"])
for k, v in d["per_config"].items():
    print("  ", k, round(v.get("ms_per_run", 0) * 1e3, 1), v.get("hbm_frac"), v.get("groups"), v.get("error"))
PY
for n in 2 4 8; do
  timeout 600 python bench.py --simulate-bands $n --no-cpu-baseline --no-per-config --no-e2e > gpurun_out/$tag/b$n.json 2> gpurun_out/$tag/b$n.err
  python -c "
import json; d=json.loads(open('gpurun_out/$tag/b$n.json').read().strip().splitlines()[-1]); print('bands $n', round(d['ms_per_step']*1e3,2), 'us', d['config']['selection'][:40], d['config']['launch'][:40])"
done

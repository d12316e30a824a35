# end-of-round check: full -m gpu suite, smoke, the default bench line, launch list of the bench's timed
# configuration and one --set full capture of the Harris kernel
tag=${1:-rf}
mkdir -p gpurun_out/$tag
( time timeout 1150 python -m pytest tests -m gpu -q -x --durations=20 ) > gpurun_out/$tag/pytest_gpu.txt 2>&1
tail -26 gpurun_out/$tag/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$tag/smoke.txt 2>&1; tail -3 gpurun_out/$tag/smoke.txt
( time timeout 1200 python bench.py ) > gpurun_out/$tag/bench.json 2> gpurun_out/$tag/bench.err
python - <<PY
import json
d = json.loads(open("gpurun_out/$tag/bench.json").read().strip().splitlines()[-1])
print("headline", round(d["ms_per_step"] * 1e3, 2), "us", round(d["roofline"]["hbm"]["frac"], 3), [(c["V"], c["TX"], c["TH"], c["PREF"]) for c in d["config"]["schedule"]], d["clocks"])
for k, v in d["per_config"].items():
    print(k, round(v.get("ms_per_run", 0) * 1e3, 1), v.get("hbm_frac"), v.get("groups"), v.get("launches_per_run"), v.get("schedule"), v.get("error"))
PY
tail -3 gpurun_out/$tag/bench.err

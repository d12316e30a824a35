mkdir -p gpurun_out/r2y
( time timeout 900 python bench.py ) > gpurun_out/r2y/bench.json 2> gpurun_out/r2y/bench.err
python - <<PY
import json
d = json.loads(open("gpurun_out/r2y/bench.json").read().strip().splitlines()[-1])
print("headline", round(d["ms_per_step"] * 1e3, 2), "us", round(d["roofline"]["hbm"]["frac"], 3), d["config"]["launch"], d["clocks"], d["gpu_launches"])
for k, v in d["per_config"].items():
    print("  ", k, round(v.get("ms_per_run", 0) * 1e3, 1), v.get("hbm_frac"), v.get("groups"), v.get("error"))
PY
tail -3 gpurun_out/r2y/bench.err

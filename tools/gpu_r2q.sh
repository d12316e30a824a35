# measured selection with varied inputs: a fresh decision cache, the bench replaying it, ncu evidence of the plans
mkdir -p gpurun_out/r2r
rm -f profiles/tuned_schedules.json
( time timeout 1500 python bench.py --retune ) > gpurun_out/r2r/bench_tune.json 2> gpurun_out/r2r/bench_tune.err
cp profiles/tuned_schedules.json gpurun_out/r2r/
( time timeout 900 python bench.py ) > gpurun_out/r2r/bench.json 2> gpurun_out/r2r/bench.err
for f in bench_tune bench; do python - <<PY
import json
d = json.loads(open("gpurun_out/r2r/$f.json").read().strip().splitlines()[-1])
print("$f headline", round(d["ms_per_step"] * 1e3, 2), "us", round(d["roofline"]["hbm"]["frac"], 3), d["config"]["selection"][:30])
for k, v in d["per_config"].items():
    print("  ", k, round(v.get("ms_per_run", 0) * 1e3, 1), v.get("hbm_frac"), v.get("groups"), v.get("error"))
PY
done
bash tools/gpu_profiles.sh r2r

# populate profiles/tuned_schedules.json (measured selection for every bench line), bring it back, then time a
# default bench run that replays the cached decisions
mkdir -p gpurun_out/r2o
rm -f profiles/tuned_schedules.json
( time timeout 1500 python bench.py --retune ) > gpurun_out/r2o/bench_tune.json 2> gpurun_out/r2o/bench_tune.err
tail -3 gpurun_out/r2o/bench_tune.err
cp profiles/tuned_schedules.json gpurun_out/r2o/ 2>/dev/null
( time timeout 1200 python bench.py ) > gpurun_out/r2o/bench.json 2> gpurun_out/r2o/bench.err
tail -3 gpurun_out/r2o/bench.err
for f in bench_tune bench; do python - <<PY
import json
d = json.loads(open("gpurun_out/r2o/$f.json").read().strip().splitlines()[-1])
print("$f headline", round(d["ms_per_step"] * 1e3, 2), "us", round(d["roofline"]["hbm"]["frac"], 3), d["config"]["selection"])
for k, v in d["per_config"].items():
    print("  ", k, round(v.get("ms_per_run", 0) * 1e3, 1), v.get("groups"), v.get("selection"), v.get("plan_s"), v.get("error"))
PY
done

# re-time the measured selection of one workload and bring the updated decision cache back
#   bash tools/gpu_retune_one.sh <workload>
wl=${1:-camera}
mkdir -p gpurun_out/retune
timeout 900 python - <<PY
import sys, json
sys.path.insert(0, ".")
import bench, pmg_inputs as PI
import paper_1909_07190_b200 as pmg
wl = PI.WORKLOADS["$wl"]
plan, how = bench.tuned_plan(pmg, pmg.Pipeline(wl.text), wl, 0, True, retune=True)
print(how, json.dumps(plan.describe().get("tune", {}))[:1500])
r = bench.measure_config("$wl", 0, 20, 5, tune=True)
print("$wl", round(r["ms_per_run"] * 1e3, 2), r["groups"], r["launches_per_run"], r["selection"])
PY
cp profiles/tuned_schedules.json gpurun_out/retune/

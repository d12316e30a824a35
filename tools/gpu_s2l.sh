# greedy measured selection: parity tests + camera timing
tag=s2l
mkdir -p gpurun_out/$tag
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "measured_selection" > gpurun_out/$tag/pytest.txt 2>&1; tail -3 gpurun_out/$tag/pytest.txt
timeout 900 python tools/sweep.py camera tune=1 > gpurun_out/$tag/tune_camera.txt 2>&1
timeout 900 python - > gpurun_out/$tag/tune_report.txt 2>&1 <<'PY'
import json, sys
sys.path.insert(0, ".")
import paper_1909_07190_b200 as pmg, pmg_inputs as PI
wl = PI.WORKLOADS["camera"]
plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=pmg.sched_opts(tune=True))
print("camera", json.dumps(plan.describe()["tune"]))
wl = PI.WORKLOADS["unsharp"]
plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=pmg.sched_opts(tune=True, fuse=False))
print("unsharp-unfused-start", json.dumps(plan.describe()["tune"]))
PY
for f in gpurun_out/$tag/*.txt; do echo $f; cat $f; done

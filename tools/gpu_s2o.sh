# measured selection with the single-group configuration grid
tag=s2o
mkdir -p gpurun_out/$tag
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "measured_selection" > gpurun_out/$tag/pytest.txt 2>&1; tail -3 gpurun_out/$tag/pytest.txt
timeout 900 python tools/sweep.py unsharp tune=1 > gpurun_out/$tag/tune_unsharp.txt 2>&1
timeout 1200 python tools/sweep.py harris tune=1 > gpurun_out/$tag/tune_harris.txt 2>&1
timeout 900 python - > gpurun_out/$tag/tune_report.txt 2>&1 <<'PY'
import json, sys
sys.path.insert(0, ".")
import paper_1909_07190_b200 as pmg, pmg_inputs as PI
for n in ["unsharp", "harris"]:
    wl = PI.WORKLOADS[n]
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=pmg.sched_opts(tune=True))
    print(n, json.dumps(plan.describe()["tune"]))
PY
for f in gpurun_out/$tag/*.txt; do echo $f; cat $f; done

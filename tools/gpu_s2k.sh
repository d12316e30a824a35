# measured selection (tune): parity test, then tuned vs model timings
tag=s2k
mkdir -p gpurun_out/$tag
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "measured_selection" > gpurun_out/$tag/pytest.txt 2>&1; tail -3 gpurun_out/$tag/pytest.txt
for w in camera unsharp harris pyramid_blend local_laplacian; do timeout 900 python tools/sweep.py $w tune=1 > gpurun_out/$tag/tune_$w.txt 2>&1; done
timeout 900 python - > gpurun_out/$tag/tune_report.txt 2>&1 <<'PY'
import json, sys
sys.path.insert(0, ".")
import paper_1909_07190_b200 as pmg, pmg_inputs as PI
for n in ["camera", "unsharp", "pyramid_blend"]:
    wl = PI.WORKLOADS[n]
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=pmg.sched_opts(tune=True))
    print(n, json.dumps(plan.describe()["tune"]))
PY
for f in gpurun_out/$tag/*.txt; do echo $f; cat $f; done

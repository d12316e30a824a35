mkdir -p gpurun_out/r2l
timeout 600 python - <<'PY'
import sys, json
sys.path.insert(0, ".")
import paper_1909_07190_b200 as pmg, pmg_inputs as PI
wl = PI.WORKLOADS["unsharp"]
plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=pmg.sched_opts(tune=True, reassoc=True))
d = plan.describe()
t = d.get("tune")
print(json.dumps(t)[:3000] if t else list(d.keys()))
PY
bash tools/bench_variants.sh r2l unsharp ";vec=1,chunks=4,rows=24,warps=1,prefetch=4" ";vec=4,chunks=1,rows=62,warps=1,prefetch=6" ";vec=4,chunks=1,rows=64,warps=1,prefetch=4"

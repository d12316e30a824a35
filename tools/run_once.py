"""Run one workload a few times (for ncu captures).  python tools/run_once.py harris [opts|auto|cached] [runs]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1909_07190_b200 as pmg  # noqa: E402
import pmg_inputs as PI  # noqa: E402
from gpu_util_bench import device_inputs  # noqa: E402

name = sys.argv[1]
spec = sys.argv[2] if len(sys.argv) > 2 and sys.argv[2] != "auto" else ""
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 3
wl = PI.WORKLOADS[name]
if spec == "cached":   # the bench's measured-selection decision (profiles/tuned_schedules.json)
    import bench
    plan, _ = bench.tuned_plan(pmg, pmg.Pipeline(wl.text), wl, 0, reassoc=True)
else:
    opts = pmg.sched_opts(**{k: int(v) for k, v in (x.split("=") for x in spec.split(","))}) if spec else None
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=opts)
ins = device_inputs(plan, wl.inputs(), 0)
outs = plan.alloc_outputs()
for _ in range(runs):
    plan.run(ins, outs)
torch.cuda.synchronize()
print(plan.describe()["kernels"])

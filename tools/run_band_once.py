"""Run one band of an N-way split a few times (for ncu).  python tools/run_band_once.py harris 8 4"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_1909_07190_b200 as pmg  # noqa: E402
import pmg_inputs as PI  # noqa: E402
from gpu_util_bench import device_inputs  # noqa: E402

name, n, b = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
wl = PI.WORKLOADS[name]
plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params)
o0, o1, i0, i1 = plan.band_rows(b, n)
ins = device_inputs(plan, wl.inputs(), 0, rows=(i0, i1))
outs = [pmg.empty_pitched((*o.shape[:-2], o1 - o0, o.shape[-1]), o.dtype) for o in plan.outputs]
for _ in range(3):
    plan.run_band(b, n, ins, outs, plan.workspace())
torch.cuda.synchronize()

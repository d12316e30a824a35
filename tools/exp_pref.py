"""Full-image and N=8 band timing for manual schedules (PREF experiment)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_1909_07190_b200 as pmg  # noqa: E402
import pmg_inputs as PI  # noqa: E402
from gpu_util_bench import device_inputs  # noqa: E402

name = sys.argv[1]
wl = PI.WORKLOADS[name]
inp = wl.inputs()
s = torch.cuda.current_stream()
for spec in sys.argv[2:]:
    kv = {k: int(v) for k, v in (x.split("=") for x in spec.split(","))}
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=pmg.sched_opts(**kv))
    res = []
    for n, b in [(1, 0), (8, 4)]:
        o0, o1, i0, i1 = plan.band_rows(b, n)
        sets = [(device_inputs(plan, inp, 0, rows=(i0, i1) if n > 1 else None),
                 [pmg.empty_pitched((*o.shape[:-2], o1 - o0, o.shape[-1]), o.dtype) for o in plan.outputs]) for _ in range(2)]
        ws = plan.workspace()
        for i in range(5):
            plan.run_band(b, n, *sets[i % 2], ws, s)
        torch.cuda.synchronize()
        graphs, cap = [], torch.cuda.Stream()
        for k in range(2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                plan.run_band(b, n, *sets[k], ws, torch.cuda.current_stream())
            graphs.append(g)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(40):
            graphs[i % 2].replay()
        e1.record(s)
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 40 * 1e3)
    print(f"{name} {spec}: full {res[0]:.1f} us, band 4/8 {res[1]:.1f} us (x{res[0]/res[1]:.2f})", flush=True)

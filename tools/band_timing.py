"""Time one row band of an N-way split on a single GPU (predicts bench.py --gpus N per-rank time)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_1909_07190_b200 as pmg  # noqa: E402
import pmg_inputs as PI  # noqa: E402
from gpu_util_bench import device_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "harris"
wl = PI.WORKLOADS[name]
plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params)
inp = wl.inputs()
s = torch.cuda.current_stream()
for n in [1, 2, 4, 8]:
    worst = 0
    for b in sorted({0, n // 2, n - 1}):
        o0, o1, i0, i1 = plan.band_rows(b, n)
        sets = []
        for _ in range(2):
            ins = device_inputs(plan, inp, 0, rows=(i0, i1) if n > 1 else None)
            outs = [pmg.empty_pitched((*o.shape[:-2], o1 - o0, o.shape[-1]), o.dtype) for o in plan.outputs]
            sets.append((ins, outs))
        ws = plan.workspace()
        for i in range(5):
            plan.run_band(b, n, *sets[i % 2], ws, s)
        torch.cuda.synchronize()
        graphs = []
        cap = torch.cuda.Stream()
        for k in range(2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                plan.run_band(b, n, *sets[k], ws, torch.cuda.current_stream())
            graphs.append(g)
        torch.cuda.synchronize()
        for i in range(5):
            graphs[i % 2].replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(50):
            graphs[i % 2].replay()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 50
        worst = max(worst, ms)
        print(f"{name} N={n} band {b}: rows [{o0},{o1}) in [{i0},{i1}) {ms*1e3:.1f} us", flush=True)
    print(f"{name} N={n}: max band {worst*1e3:.1f} us -> projected {wl.params['W']*wl.params['H']/worst/1e3:.0f} Mpx/s total", flush=True)

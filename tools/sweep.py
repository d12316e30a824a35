"""Time a workload under a list of manual schedules (device time per pipeline run, CUDA events, 2 rotating
buffer sets).  Used to calibrate the selector against measurement (§6.1 weight fitting).

    python tools/sweep.py harris "vec=4,chunks=1,rows=32,warps=4,prefetch=4" "vec=2,chunks=2,rows=64,warps=4,prefetch=4"
    python tools/sweep.py harris grid
"""
import itertools
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1909_07190_b200 as pmg  # noqa: E402
import pmg_inputs as PI  # noqa: E402
from gpu_util_bench import device_inputs  # noqa: E402


def time_plan(plan, inputs_np, steps=20):
    sets = [(device_inputs(plan, inputs_np, 0), plan.alloc_outputs()) for _ in range(2)]
    ws = plan.workspace()
    s = torch.cuda.current_stream()
    for i in range(3):
        plan.run(*sets[i % 2], ws, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(steps):
        plan.run(*sets[i % 2], ws, s)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    name = sys.argv[1]
    wl = PI.WORKLOADS[name]
    if len(sys.argv) > 2 and sys.argv[2].startswith("W="):
        W = int(sys.argv[2][2:].split("x")[0]); H = int(sys.argv[2].split("x")[1])
        wl = PI.small(name, W, H)
        specs = sys.argv[3:]
    else:
        specs = sys.argv[2:]
    if specs == ["grid"]:
        specs = [f"vec={v},chunks={tx},rows={th},warps={nw},prefetch={pf}"
                 for v, tx, th, nw, pf in itertools.product([2, 4], [1, 2], [8, 16, 24, 32, 64], [1, 2], [4])]
    inputs_np = wl.inputs()
    pipe = pmg.Pipeline(wl.text)
    px = wl.params["W"] * wl.params["H"]
    nbytes = None
    for spec in ["auto"] + specs:
        try:
            # gos=0.1.1.2 gives group_of_stage (one group id per stage, '.'-separated)
            kv = {k: ([int(q) for q in v.split(".")] if k == "gos" else int(v))
                  for k, v in (x.split("=") for x in spec.split(","))} if spec != "auto" else None
            if kv and "gos" in kv:
                kv["group_of_stage"] = kv.pop("gos")
            opts = None if spec == "auto" else pmg.sched_opts(**kv)
            plan = pmg.Plan(pipe, wl.params, opts=opts)
            if nbytes is None:
                nbytes = sum(int(torch.tensor(io.shape).prod()) * pmg._binding.DTYPE_SIZE[io.dtype]
                             for io in plan.inputs + plan.outputs)
            ms = time_plan(plan, inputs_np)
            d = plan.describe()
            ks = [(k["regs"], k["spill_stores"], k["blocks_per_sm"]) for k in d["kernels"]]
            print(json.dumps({"spec": spec, "ms": round(ms, 4), "Mpx/s": round(px / ms / 1e3, 1),
                              "GB/s": round(nbytes / ms / 1e6, 1), "kernels(regs,spill,blk/SM)": ks[:4],
                              "nk": len(ks)}), flush=True)
        except Exception as e:
            print(json.dumps({"spec": spec, "error": str(e)[:300]}), flush=True)


if __name__ == "__main__":
    main()

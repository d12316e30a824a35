"""Small runs of the hot path for compute-sanitizer (tests/test_gpu_sanitizer.py): whole images (interior,
x-edge and border kernels), row bands on buffers holding exactly the band's input rows, and a batch.  Run with
PYTORCH_NO_CUDA_MEMORY_CACHING=1 so every tensor is its own cudaMalloc (memcheck sees accesses past a buffer).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [harris|camera|ll|unsharp]...
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1909_07190_b200 as pmg  # noqa: E402
import pmg_inputs as PI  # noqa: E402
from gpu_util_bench import device_inputs  # noqa: E402

CASES = {
    "harris": PI.small("harris", 512, 211),          # x-edge kernel (W % 4 == 0), border rows, 5 bands
    "unsharp": PI.small("unsharp", 300, 130),        # no x-edge kernel (W % 4 != 0): x-border tiles
    "camera": PI.small("camera", 264, 130),          # phase-split denoise + demosaic, gathers
    "ll": PI.Workload("ll", "local_laplacian_J4K4.pmg", {"W": 96, "H": 64}, 1005),
}


def main(names):
    for name in names:
        wl = CASES[name]
        inp = wl.inputs("structured") if name == "ll" else wl.inputs()
        plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params)
        outs = plan.run(device_inputs(plan, inp, 0))
        torch.cuda.synchronize()
        nb = 5 if name == "harris" else 3
        bplan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=pmg.sched_opts(bands=nb))
        for b in range(nb):
            o_r0, o_r1, i_r0, i_r1 = bplan.band_rows(b, nb)
            ins = device_inputs(bplan, inp, 0, rows=(i_r0, i_r1))
            bouts = [pmg.empty_pitched((*o.shape[:-2], o_r1 - o_r0, o.shape[-1]), o.dtype, "cuda:0") for o in bplan.outputs]
            bplan.run_band(b, nb, ins, bouts, bplan.workspace())
            torch.cuda.synchronize()
            for o, t, full in zip(bplan.outputs, bouts, outs):
                assert torch.equal(t.contiguous(), full[..., o_r0:o_r1, :].contiguous()), (name, b)
        print(f"[sanitize] {name}: whole image + {nb} bands ok")


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))

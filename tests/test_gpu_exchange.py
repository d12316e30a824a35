"""GPU parity of the halo-exchange band mode: every band of an image runs in this process with
pmg_run_band_groups on exactly its geometry's input rows, the halo rows of each workspace stage are copied from
the owning band's workspace after the producing group (dist.run_bands_exchange_local), and the stitched liveout
rows must equal the whole-image oracle bit for bit.  Pyramids (local Laplacian, pyramid blend) exchange at every
level; single-group pipelines (Harris) exchange nothing and read only their own rows plus the input halo."""
import numpy as np
import pytest

import pmg_inputs as PI
from gpu_util import to_device, to_numpy
from oracle import evaluate

pytestmark = pytest.mark.gpu

import paper_1909_07190_b200 as pmg  # noqa: E402
from paper_1909_07190_b200.dist import run_bands_exchange_local  # noqa: E402

CASES = {   # (camera bands: recompute geometry in test_gpu_fullsize.py; its exchange rows follow the same code)
    "pb_small": (lambda: PI.Workload("pb", "pyramid_blend_J3.pmg", {"W": 97, "H": 63}, 1006), 4, "structured"),
    "harris": (lambda: PI.small("harris", 300, 211), 5, None),
    "local_laplacian_full": (lambda: PI.WORKLOADS["local_laplacian"], 8, "structured"),
}


def run_exchange(wl, nb, inp):
    import torch
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=pmg.sched_opts(bands=nb))
    geoms = [plan.band_exchange(b, nb) for b in range(nb)]
    ins, outs, wss = [], [], []
    for b, g in enumerate(geoms):
        r0, r1 = g["in"]
        ins.append([to_device(inp[io.name] if io.is_table else inp[io.name][..., r0:r1, :], io.dtype,
                              pitched=not io.is_table) for io in plan.inputs])
        o0, o1 = g["out"]
        outs.append([pmg.empty_pitched((*o.shape[:-2], o1 - o0, o.shape[-1]), o.dtype) for o in plan.outputs])
        wss.append(torch.zeros(max(16, plan.workspace_bytes), dtype=torch.uint8, device="cuda:0"))
    run_bands_exchange_local(plan, nb, ins, outs, wss)
    torch.cuda.synchronize()
    got = {}
    for k, o in enumerate(plan.outputs):
        got[o.name] = np.concatenate([to_numpy(outs[b][k]) for b in range(nb)], axis=-2)
    return got, geoms, plan


@pytest.mark.parametrize("case", list(CASES))
def test_halo_exchange_bands_equal_oracle(case):
    mk, nb, variant = CASES[case]
    wl = mk()
    inp = wl.inputs(variant) if variant else wl.inputs()
    exp = evaluate(wl.text, wl.params, inp)
    got, geoms, plan = run_exchange(wl, nb, inp)
    for name, e in exp.items():
        assert got[name].shape == e.shape
        neq = int(np.count_nonzero(got[name].view(np.uint8) != e.view(np.uint8)))
        assert neq == 0, f"{case}: {neq} bytes of {name} differ from the oracle"
    if case.startswith(("pb", "local")):
        assert any(g["recv"] for g in geoms), "a pyramid must exchange halo rows"
        # the band reads far fewer input rows than the cumulative-halo recompute needs
        mid = nb // 2
        _, _, i0, i1 = plan.band_rows(mid, nb)
        assert geoms[mid]["in"][1] - geoms[mid]["in"][0] < i1 - i0

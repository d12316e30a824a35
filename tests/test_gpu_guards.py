"""Out-of-bounds checks of our own (compute-sanitizer is closed on this GPU pool): every device buffer the hot
path touches is surrounded by poisoned guard zones, and the runs must neither read nor write them.

* inputs: each image (whole, or exactly a band's input rows) sits inside a larger allocation whose guard rows
  above / below every plane and columns past the 16-byte-aligned width hold poison (NaN for f32, all-ones for
  integers); a kernel that READ a guard element would carry the poison into an output, so outputs must equal
  the oracle / the whole-image run bit for bit;
* outputs: the same layout filled with a sentinel; guard rows and columns past the aligned width must still hold
  it after the run (no out-of-bounds WRITE);
* workspace: the plan's workspace sits between two 4 KB sentinel zones that must be untouched.

Cases cover the interior, x-edge and border kernels (Harris 512 wide: x-edge; unsharp 300 wide: x-border
tiles), gathers and phase splits (camera), scaled streams across pyramid levels (4-level local Laplacian), and
row bands holding exactly their input rows (band-mode clamping)."""
import numpy as np
import pytest

import pmg_inputs as PI
from gpu_util import compare, to_device, to_numpy
from oracle import evaluate

pytestmark = pytest.mark.gpu

import paper_1909_07190_b200 as pmg  # noqa: E402

G = 24          # guard rows above and below every plane
GC = 64         # guard bytes past the 16-byte-aligned width

CASES = {
    "harris": (PI.small("harris", 512, 211), 5),
    "unsharp": (PI.small("unsharp", 300, 130), 3),
    "camera": (PI.small("camera", 264, 130), 3),
    "ll": (PI.Workload("ll", "local_laplacian_J4K4.pmg", {"W": 96, "H": 64}, 1005), 3),
}


def _poison(dtype: str):
    return float("nan") if dtype == "f32" else -1


def guarded(arr_shape, dtype, fill, device="cuda:0"):
    """(storage, view): view has arr_shape, planes and rows surrounded by guard zones holding `fill`."""
    import torch
    esz = pmg._binding.DTYPE_SIZE[dtype]
    *planes, rows, w = arr_shape
    wa = (w * esz + 15) // 16 * 16 // esz
    wp = wa + GC // esz
    tdt = pmg.pipeline._torch_dtype(dtype)
    if tdt == torch.uint16:
        tdt = torch.int16
    store = torch.full((*planes, rows + 2 * G, wp), fill, dtype=tdt, device=device)
    view = store[..., G:G + rows, :w]
    if pmg.pipeline._torch_dtype(dtype) == torch.uint16:
        view = view.view(torch.uint16)
    return store, view


def guards_intact(store, rows, w, esz, fill) -> bool:
    import torch
    wa = (w * esz + 15) // 16 * 16 // esz
    s = store.view(torch.int16) if store.dtype == torch.uint16 else store
    top, bot, right = s[..., :G, :], s[..., G + rows:, :], s[..., G:G + rows, wa:]
    def same(t):
        if t.numel() == 0:
            return True
        if isinstance(fill, float) and np.isnan(fill):
            return bool(torch.isnan(t).all())
        return bool((t == fill).all())
    return same(top) and same(bot) and same(right)


def run_guarded(plan, inp, rows=None, band=None):
    """One run (whole image, or band (b, n) on exactly its input rows) with guarded buffers; returns outputs as
    numpy and asserts every guard zone is intact."""
    import torch
    ins, stores = [], []
    for io in plan.inputs:
        arr = inp[io.name]
        if io.is_table:
            ins.append(to_device(arr, io.dtype, pitched=False))
            continue
        if rows is not None:
            arr = arr[..., rows[0]:rows[1], :]
        st, v = guarded(arr.shape, io.dtype, _poison(io.dtype))
        src = torch.from_numpy(np.ascontiguousarray(arr).view(np.int16) if arr.dtype == np.uint16 else np.ascontiguousarray(arr))
        (v.view(torch.int16) if v.dtype == torch.uint16 else v).copy_(src.to("cuda:0"))
        ins.append(v)
        stores.append((st, arr.shape[-2], arr.shape[-1], pmg._binding.DTYPE_SIZE[io.dtype], _poison(io.dtype)))
    outs, ostores = [], []
    for o in plan.outputs:
        shape = o.shape if band is None else (*o.shape[:-2], band[1] - band[0], o.shape[-1])
        sent = 12345.0 if o.dtype == "f32" else 77
        st, v = guarded(shape, o.dtype, sent)
        outs.append(v)
        ostores.append((st, shape[-2], shape[-1], pmg._binding.DTYPE_SIZE[o.dtype], sent))
    wsn = max(16, plan.workspace_bytes)
    ws = torch.full((wsn + 8192,), 0x5A, dtype=torch.uint8, device="cuda:0")
    wsv = ws[4096:4096 + wsn]
    if band is None:
        plan.run(ins, outs, wsv)
    else:
        plan.run_band(band[2], band[3], ins, outs, wsv)
    torch.cuda.synchronize()
    for st in stores:
        assert guards_intact(*st), "an input guard zone changed"
    for st in ostores:
        assert guards_intact(*st), "a kernel wrote outside its output rows / aligned width"
    assert bool((ws[:4096] == 0x5A).all()) and bool((ws[4096 + wsn:] == 0x5A).all()), "workspace overrun"
    return [to_numpy(v) for v in outs]


@pytest.mark.parametrize("name", list(CASES))
def test_guard_zones_whole_image_and_bands(name):
    wl, nb = CASES[name]
    inp = wl.inputs("structured") if name == "ll" else wl.inputs()
    exp = evaluate(wl.text, wl.params, inp)
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params)
    got = run_guarded(plan, inp)
    for o, g in zip(plan.outputs, got):
        neq, _ = compare(g, exp[o.name], float_tol=1e-4, rel_range=1e-5 if name == "harris" else None)
        assert neq == 0, f"{name}: {neq} outputs differ from the oracle with guarded inputs"
    bplan = plan            # the same kernels run the bands (one compile per case)
    for b in range(nb):
        o_r0, o_r1, i_r0, i_r1 = bplan.band_rows(b, nb)
        res = run_guarded(bplan, inp, rows=(i_r0, i_r1), band=(o_r0, o_r1, b, nb))
        for o, g in zip(bplan.outputs, res):
            e = exp[o.name][..., o_r0:o_r1, :]
            assert np.array_equal(g.view(np.uint8), e.view(np.uint8)), f"{name}: band {b} of {nb} differs"

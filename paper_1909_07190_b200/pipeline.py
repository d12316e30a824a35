"""Thin Python API over the C ABI: Pipeline (parse / inspect / schedule / emit), Plan (compile for a device
and run on torch tensors).  Names follow include/pmg.h and the paper (§2.2, §4-§6)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _binding as B

TORCH_DTYPES = None


def _torch_dtype(name):
    import torch
    return {"f32": torch.float32, "i32": torch.int32, "i16": torch.int16, "u16": torch.uint16, "u8": torch.uint8}[name]


@dataclass
class IO:
    name: str
    dtype: str
    shape: tuple
    is_table: bool


def gpu_spec(name: str = "b200") -> B.GpuSpec:
    s = B.GpuSpec()
    B.check(B.lib.pmg_gpu_spec_preset(name.encode(), C.byref(s)))
    return s


def query_gpu_spec(device: int = 0, measured_bw_gbs: float = 0.0) -> B.GpuSpec:
    s = B.GpuSpec()
    B.check(B.lib.pmg_gpu_spec_query(device, measured_bw_gbs, C.byref(s)))
    return s


def weights(name: str = "b200") -> B.Weights:
    w = B.Weights()
    B.check(B.lib.pmg_weights_preset(name.encode(), C.byref(w)))
    return w


def sched_opts(group_of_stage=None, vec=-1, chunks=-1, smem_chunks=-1, rows=-1, warps=-1, prefetch=-1, tx_size=-1,
               budget=0, fuse=True, regcap=0, probe=True, cost_model=0, bands=0, inline=True, tune=False,
               time_per_iter=None, reassoc=False, border_rows=0) -> B.SchedOpts:
    o = B.SchedOpts()
    B.lib.pmg_sched_opts_default(C.byref(o))
    o.vec, o.chunks, o.smem_chunks, o.rows, o.warps, o.prefetch, o.tx_size = (
        vec, chunks, smem_chunks, rows, warps, prefetch, tx_size)
    o.budget = budget
    o.fuse = 1 if fuse else 0
    o.regcap = regcap
    o.probe = 1 if probe else 0
    o.cost_model = cost_model          # 0: B200 time estimate, 1: Alg. 2 weighted sum
    o.bands = bands                    # expected row-band split (the estimate counts one band's tiles)
    o.no_inline = 0 if inline else 1   # substitute data-expanding stages into their readers
    o.tune = 1 if tune else 0          # measured selection among the DP schedule and its neighbour merges
    o.reassoc = 1 if reassoc else 0    # separable rank-1 stencils + fma contraction (f32 rounding differs)
    o.border_rows = border_rows        # border-tile rows (TH_b); 0 = automatic
    if time_per_iter is not None:       # measured TimePerIter per stage (Pipeline.profile_stages), Alg. 2 input
        tarr = (C.c_double * len(time_per_iter))(*time_per_iter)
        o._keep_tpi = tarr
        o.time_per_iter = C.cast(tarr, C.POINTER(C.c_double))
    if group_of_stage is not None:
        arr = (C.c_int32 * len(group_of_stage))(*group_of_stage)
        o._keep = arr                      # keep the array alive with the struct
        o.group_of_stage = C.cast(arr, C.POINTER(C.c_int32))
    return o


class Pipeline:
    """A parsed, validated stage DAG (immutable)."""

    def __init__(self, text: str):
        h = C.c_void_p()
        data = text.encode()
        B.check(B.lib.pmg_pipeline_parse(data, len(data), C.byref(h)))
        self._h = h
        self.text = text

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and getattr(B, "lib", None) is not None:   # (the module may be torn down at interpreter exit)
            B.lib.pmg_pipeline_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def _names(self, count_fn, name_fn):
        n = count_fn(self._h)
        out = []
        for i in range(n):
            buf = C.create_string_buffer(256)
            B.check(name_fn(self._h, i, buf, 256))
            out.append(buf.value.decode())
        return out

    @property
    def params(self):
        return self._names(B.lib.pmg_pipeline_num_params, B.lib.pmg_pipeline_param_name)

    @property
    def stages(self):
        return self._names(B.lib.pmg_pipeline_num_stages, B.lib.pmg_pipeline_stage_name)

    def param_values(self, params: dict):
        missing = [p for p in self.params if p not in params]
        if missing:
            raise B.PmgError(-9, f"missing parameter values {missing}")
        return B.i64arr(params[p] for p in self.params)

    def io(self, params: dict, is_output: bool):
        arr, n = self.param_values(params)
        out = []
        for i in range(B.lib.pmg_pipeline_num_io(self._h, int(is_output))):
            d = B.IODesc()
            B.check(B.lib.pmg_pipeline_io(self._h, int(is_output), i, arr, n, C.byref(d)))
            out.append(IO(d.name.decode(), B.DTYPES[d.dtype], tuple(d.extent[:d.ndim]), bool(d.is_table)))
        return out

    def inputs(self, params):
        return self.io(params, False)

    def outputs(self, params):
        return self.io(params, True)

    def describe(self, params: dict) -> dict:
        arr, n = self.param_values(params)
        return B.call_json(B.lib.pmg_pipeline_describe, self._h, arr, n)

    def inlined(self, params: dict) -> dict:
        """{"inlined": [stage names], "text": pipeline text} after substituting data-expanding stages."""
        arr, n = self.param_values(params)
        return B.call_json(B.lib.pmg_pipeline_inlined, self._h, arr, n)

    def rewritten(self, params: dict, opts=None) -> dict:
        """{"factored", "inlined", "split", "text"}: the pipeline text a plan made with `opts` schedules."""
        arr, n = self.param_values(params)
        return B.call_json(B.lib.pmg_pipeline_rewritten, self._h, arr, n, _ref(opts))

    def profile_stages(self, params: dict, device: int = 0) -> dict:
        """On-device TimePerIter of every stage (each stage alone as one kernel)."""
        import json as _json
        arr, n = self.param_values(params)
        cap = 1 << 20                       # one call: the profile runs kernels, so no size-query round trip
        buf = C.create_string_buffer(cap)
        need = C.c_size_t(0)
        B.check(B.lib.pmg_profile_stages(self._h, arr, n, device, buf, cap, C.byref(need)))
        return _json.loads(buf.value.decode())

    def schedule(self, params: dict, spec=None, weights_=None, opts=None) -> dict:
        arr, n = self.param_values(params)
        return B.call_json(B.lib.pmg_schedule, self._h, arr, n, _ref(spec), _ref(weights_), _ref(opts))

    def analyze_group(self, params: dict, stages, tile, block, frac_reg=0.0, tx_size=128, regs_per_stage=16,
                      spec=None, weights_=None) -> dict:
        arr, n = self.param_values(params)
        t = (C.c_int32 * 3)(*tile)
        b = (C.c_int32 * 3)(*block)
        return B.call_json(B.lib.pmg_analyze_group, self._h, arr, n, ",".join(stages).encode(), t, b, float(frac_reg),
                           tx_size, regs_per_stage, _ref(spec), _ref(weights_))

    def band_rows(self, params: dict, band: int, nbands: int, spec=None, weights_=None, opts=None):
        """(out_r0, out_r1, in_r0, in_r1) of row band `band` of `nbands` (host-only geometry)."""
        arr, n = self.param_values(params)
        v = [C.c_int64() for _ in range(4)]
        B.check(B.lib.pmg_band_rows_host(self._h, arr, n, _ref(spec), _ref(weights_), _ref(opts), band, nbands,
                                         *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def band_exchange(self, params: dict, band: int, nbands: int, spec=None, weights_=None, opts=None) -> dict:
        """Halo-exchange band geometry (host only): own rows per group, workspace slots, sends / receives."""
        arr, n = self.param_values(params)
        return B.call_json(B.lib.pmg_band_exchange_host, self._h, arr, n, _ref(spec), _ref(weights_), _ref(opts),
                           band, nbands)

    def emit(self, params: dict, spec=None, weights_=None, opts=None) -> dict:
        arr, n = self.param_values(params)
        return B.call_json(B.lib.pmg_emit, self._h, arr, n, _ref(spec), _ref(weights_), _ref(opts))

    def precompile(self, params: dict, out_dir: str = "", spec=None, weights_=None, opts=None) -> dict:
        arr, n = self.param_values(params)
        return B.call_json(B.lib.pmg_precompile, self._h, arr, n, _ref(spec), _ref(weights_), _ref(opts),
                           out_dir.encode())


def _ref(x):
    return C.byref(x) if x is not None else None


def _buf(t) -> B.Buf:
    """torch tensor (1-3 dims, planar [c][y][x], x contiguous) -> pmg_buf."""
    if t.dim() == 0 or t.stride(-1) != 1:
        raise B.PmgError(-9, "tensors must have a contiguous last (x) dimension")
    esz = t.element_size()
    rp = t.stride(-2) * esz if t.dim() >= 2 else t.shape[-1] * esz
    pp = t.stride(-3) * esz if t.dim() >= 3 else rp * (t.shape[-2] if t.dim() >= 2 else 1)
    return B.Buf(C.c_void_p(t.data_ptr()), rp, pp)


def empty_pitched(shape, dtype: str, device="cuda", frames: int = 0):
    """Device tensor whose row pitch is a multiple of 16 bytes (the ABI's alignment rule); returns a view."""
    import torch
    esz = B.DTYPE_SIZE[dtype]
    w = shape[-1]
    wp = ((w * esz + 15) // 16 * 16) // esz
    full = tuple(shape[:-1]) + (wp,)
    if frames:
        full = (frames,) + full
    t = torch.empty(full, dtype=_torch_dtype(dtype), device=device)
    return t[..., :w]


class Plan:
    """A pipeline bound to parameter values, a device and a schedule; kernels compiled for sm_100a."""

    def __init__(self, pipeline: Pipeline, params: dict, device: int = 0, spec=None, weights_=None, opts=None):
        self.pipeline = pipeline
        self.params = dict(params)
        self.device = device
        arr, n = pipeline.param_values(params)
        h = C.c_void_p()
        B.check(B.lib.pmg_plan_create(pipeline.handle, arr, n, device, _ref(spec), _ref(weights_), _ref(opts),
                                      C.byref(h)))
        self._h = h
        self.inputs = pipeline.inputs(params)
        self.outputs = pipeline.outputs(params)
        ws = C.c_size_t(0)
        B.check(B.lib.pmg_plan_workspace_bytes(h, C.byref(ws)))
        self.workspace_bytes = ws.value
        self._ws = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and getattr(B, "lib", None) is not None:   # (the module may be torn down at interpreter exit)
            B.lib.pmg_plan_destroy(h)
            self._h = None

    def describe(self) -> dict:
        return B.call_json(B.lib.pmg_plan_describe, self._h)

    @property
    def num_kernels(self) -> int:
        return B.lib.pmg_plan_num_kernels(self._h)

    @property
    def last_launches(self) -> int:
        """kernels launched by the most recent run call (interior + border kernels of every group)"""
        return B.lib.pmg_plan_last_launches(self._h)

    def workspace(self, frames: int = 1):
        import torch
        need = max(16, self.workspace_bytes * frames)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{self.device}")
        return self._ws

    def alloc_outputs(self, frames: int = 0):
        return [empty_pitched(o.shape, o.dtype, f"cuda:{self.device}", frames) for o in self.outputs]

    def _stream(self, stream):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return C.c_void_p(s.cuda_stream)

    def run(self, inputs, outputs=None, workspace=None, stream=None):
        """inputs: tensors in pmg_pipeline_io order (images then tables); returns the output tensors."""
        if outputs is None:
            outputs = self.alloc_outputs()
        ib = (B.Buf * max(1, len(inputs)))(*[_buf(t) for t in inputs])
        ob = (B.Buf * max(1, len(outputs)))(*[_buf(t) for t in outputs])
        ws = workspace if workspace is not None else self.workspace()
        B.check(B.lib.pmg_run(self._h, ib, len(inputs), ob, len(outputs), C.c_void_p(ws.data_ptr()),
                              self._stream(stream)))
        return outputs

    def run_batch(self, inputs, outputs, workspace=None, stream=None):
        """Frame-major batches: every image/output tensor has a leading frame dim; tables are shared."""
        nframes = outputs[0].shape[0]
        ib, ifs = [], []
        for t, io in zip(inputs, self.inputs):
            if io.is_table:
                ib.append(_buf(t))
                ifs.append(0)
            else:
                ib.append(_buf(t[0]))
                ifs.append(t.stride(0) * t.element_size())
        ob = [_buf(t[0]) for t in outputs]
        ofs = [t.stride(0) * t.element_size() for t in outputs]
        ws = workspace if workspace is not None else self.workspace(nframes)
        ia, _ = B.i64arr(ifs)
        oa, _ = B.i64arr(ofs)
        B.check(B.lib.pmg_run_batch(self._h, nframes, (B.Buf * len(ib))(*ib), ia, len(ib), (B.Buf * len(ob))(*ob), oa,
                                    len(ob), C.c_void_p(ws.data_ptr()), self._stream(stream)))
        return outputs

    def band_rows(self, band: int, nbands: int):
        v = [C.c_int64() for _ in range(4)]
        B.check(B.lib.pmg_band_rows(self._h, band, nbands, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)   # out_r0, out_r1, in_r0, in_r1

    def band_exchange(self, band: int, nbands: int) -> dict:
        """Halo-exchange band geometry of this plan (pmg_band_exchange)."""
        return B.call_json(B.lib.pmg_band_exchange, self._h, band, nbands)

    def run_band_groups(self, band: int, nbands: int, g0: int, g1: int, inputs, outputs, workspace, stream=None):
        """Halo-exchange band mode: groups [g0, g1) of band `band` (inputs hold the geometry's "in" rows)."""
        ib = (B.Buf * max(1, len(inputs)))(*[_buf(t) for t in inputs])
        ob = (B.Buf * max(1, len(outputs)))(*[_buf(t) for t in outputs])
        B.check(B.lib.pmg_run_band_groups(self._h, band, nbands, g0, g1, ib, len(inputs), ob, len(outputs),
                                          C.c_void_p(workspace.data_ptr()), self._stream(stream)))
        return outputs

    def run_band(self, band: int, nbands: int, inputs, outputs, workspace=None, stream=None):
        """inputs[i] holds image rows [in_r0, in_r1) (tables whole); outputs hold rows [out_r0, out_r1)."""
        ib = (B.Buf * max(1, len(inputs)))(*[_buf(t) for t in inputs])
        ob = (B.Buf * max(1, len(outputs)))(*[_buf(t) for t in outputs])
        ws = workspace if workspace is not None else self.workspace()
        B.check(B.lib.pmg_run_band(self._h, band, nbands, ib, len(inputs), ob, len(outputs), C.c_void_p(ws.data_ptr()),
                                   self._stream(stream)))
        return outputs


    def run_host(self, host_inputs, host_outputs, dev_inputs, dev_outputs, chunks: int = 8, workspace=None,
                 stream=None):
        """End-to-end run from host tensors (pinned CPU tensors for asynchronous copies) through full-size device
        staging tensors; `chunks` row bands pipeline copy-in, compute and copy-out (pmg_run_host)."""
        hi = (B.Buf * max(1, len(host_inputs)))(*[_buf(t) for t in host_inputs])
        ho = (B.Buf * max(1, len(host_outputs)))(*[_buf(t) for t in host_outputs])
        di = (B.Buf * max(1, len(dev_inputs)))(*[_buf(t) for t in dev_inputs])
        do = (B.Buf * max(1, len(dev_outputs)))(*[_buf(t) for t in dev_outputs])
        ws = workspace if workspace is not None else self.workspace()
        B.check(B.lib.pmg_run_host(self._h, hi, len(host_inputs), ho, len(host_outputs), di, do,
                                   C.c_void_p(ws.data_ptr()), int(chunks), self._stream(stream)))
        return host_outputs


def selftest_shuffle(device: int = 0) -> int:
    v = C.c_int32(-1)
    B.check(B.lib.pmg_selftest_shuffle(device, C.byref(v)))
    return v.value

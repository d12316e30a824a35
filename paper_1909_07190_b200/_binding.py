"""ctypes binding of include/pmg.h — argument marshalling only (every step of the path runs in libpmg.so
and its sm_100a kernels).  PyTorch supplies device memory and streams.  There is no CPU fallback: if the
native library is missing, importing this module raises."""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

HERE = Path(__file__).resolve().parent
LIBPATH = HERE / "libpmg.so"

if not LIBPATH.exists():
    raise ImportError(f"{LIBPATH} is missing: build it with `python -m paper_1909_07190_b200.build_lib` "
                      "(or __graft_entry__.build()); there is no fallback path")
# libpmg.so resolves libnvrtc.so.12 at load time.  PyTorch brings its own NVRTC (12.8) and every GPU process
# imports torch, so load torch first: the same NVRTC / ptxas then compiles the kernels in every process (the
# host-only build() and the GPU runs), and the cubin cache, register counts and selector decisions agree.
try:
    import torch  # noqa: F401
except Exception:  # pragma: no cover - torch is part of the image
    pass
lib = C.CDLL(str(LIBPATH))

PMG_OK = 0
STATUS = {0: "PMG_OK", -1: "PMG_ERR_PARSE", -2: "PMG_ERR_INVALID", -3: "PMG_ERR_UNSUPPORTED",
          -4: "PMG_ERR_INFEASIBLE", -5: "PMG_ERR_SHAPE", -6: "PMG_ERR_CUDA", -7: "PMG_ERR_NVRTC",
          -8: "PMG_ERR_OOM", -9: "PMG_ERR_ARG"}
DTYPES = {1: "u8", 2: "u16", 3: "i16", 4: "i32", 5: "f32"}
DTYPE_SIZE = {"u8": 1, "u16": 2, "i16": 2, "i32": 4, "f32": 4}


class PmgError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class IODesc(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("dtype", C.c_int32), ("ndim", C.c_int32), ("is_table", C.c_int32),
                ("reserved", C.c_int32), ("extent", C.c_int64 * 3)]


class Buf(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("row_pitch_bytes", C.c_int64), ("plane_pitch_bytes", C.c_int64)]


class GpuSpec(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("nsms", C.c_int32), ("cores_per_sm", C.c_int32),
                ("max_warps_per_sm", C.c_int32), ("max_tb_per_sm", C.c_int32), ("regs_per_sm", C.c_int32),
                ("max_regs_per_thread", C.c_int32), ("max_threads_per_sm", C.c_int32), ("warp_size", C.c_int32),
                ("shmem_per_sm", C.c_int64), ("max_shmem_per_tb", C.c_int64), ("gl_mem_bw", C.c_double),
                ("gl_tx_size", C.c_int32 * 2), ("l2_bytes", C.c_int64), ("sm_clock_hz", C.c_double)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["name"] = self.name.decode()
        d["gl_tx_size"] = list(self.gl_tx_size)
        return d


class Weights(C.Structure):
    _fields_ = [("w", C.c_double * 7)]


class SchedOpts(C.Structure):
    _fields_ = [("group_of_stage", C.POINTER(C.c_int32)), ("vec", C.c_int32), ("chunks", C.c_int32),
                ("smem_chunks", C.c_int32), ("rows", C.c_int32), ("warps", C.c_int32), ("prefetch", C.c_int32),
                ("tx_size", C.c_int32), ("budget", C.c_int32), ("fuse", C.c_int32), ("regcap", C.c_int32),
                ("probe", C.c_int32), ("cost_model", C.c_int32), ("bands", C.c_int32), ("no_inline", C.c_int32),
                ("tune", C.c_int32), ("reassoc", C.c_int32), ("time_per_iter", C.POINTER(C.c_double)),
                ("border_rows", C.c_int32), ("reserved2", C.c_int32)]


P = C.c_void_p
I64P = C.POINTER(C.c_int64)
_sig = {
    "pmg_last_error": (C.c_char_p, []),
    "pmg_version": (C.c_char_p, []),
    "pmg_pipeline_parse": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(P)]),
    "pmg_pipeline_destroy": (None, [P]),
    "pmg_pipeline_num_params": (C.c_int, [P]),
    "pmg_pipeline_param_name": (C.c_int, [P, C.c_int, C.c_char_p, C.c_size_t]),
    "pmg_pipeline_num_stages": (C.c_int, [P]),
    "pmg_pipeline_stage_name": (C.c_int, [P, C.c_int, C.c_char_p, C.c_size_t]),
    "pmg_pipeline_num_io": (C.c_int, [P, C.c_int]),
    "pmg_pipeline_io": (C.c_int, [P, C.c_int, C.c_int, I64P, C.c_int, C.POINTER(IODesc)]),
    "pmg_pipeline_describe": (C.c_int, [P, I64P, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "pmg_gpu_spec_preset": (C.c_int, [C.c_char_p, C.POINTER(GpuSpec)]),
    "pmg_gpu_spec_query": (C.c_int, [C.c_int, C.c_double, C.POINTER(GpuSpec)]),
    "pmg_weights_preset": (C.c_int, [C.c_char_p, C.POINTER(Weights)]),
    "pmg_sched_opts_default": (None, [C.POINTER(SchedOpts)]),
    "pmg_profile_stages": (C.c_int, [P, I64P, C.c_int, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "pmg_schedule": (C.c_int, [P, I64P, C.c_int, C.POINTER(GpuSpec), C.POINTER(Weights), C.POINTER(SchedOpts),
                               C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "pmg_analyze_group": (C.c_int, [P, I64P, C.c_int, C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                    C.c_double, C.c_int32, C.c_int32, C.POINTER(GpuSpec), C.POINTER(Weights),
                                    C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "pmg_emit": (C.c_int, [P, I64P, C.c_int, C.POINTER(GpuSpec), C.POINTER(Weights), C.POINTER(SchedOpts),
                           C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "pmg_precompile": (C.c_int, [P, I64P, C.c_int, C.POINTER(GpuSpec), C.POINTER(Weights), C.POINTER(SchedOpts),
                                 C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "pmg_plan_create": (C.c_int, [P, I64P, C.c_int, C.c_int, C.POINTER(GpuSpec), C.POINTER(Weights),
                                  C.POINTER(SchedOpts), C.POINTER(P)]),
    "pmg_plan_destroy": (None, [P]),
    "pmg_plan_describe": (C.c_int, [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "pmg_plan_workspace_bytes": (C.c_int, [P, C.POINTER(C.c_size_t)]),
    "pmg_plan_num_kernels": (C.c_int, [P]),
    "pmg_plan_last_launches": (C.c_int, [P]),
    "pmg_run": (C.c_int, [P, C.POINTER(Buf), C.c_int, C.POINTER(Buf), C.c_int, C.c_void_p, C.c_void_p]),
    "pmg_run_batch": (C.c_int, [P, C.c_int, C.POINTER(Buf), I64P, C.c_int, C.POINTER(Buf), I64P, C.c_int,
                                C.c_void_p, C.c_void_p]),
    "pmg_band_rows": (C.c_int, [P, C.c_int, C.c_int, I64P, I64P, I64P, I64P]),
    "pmg_band_rows_host": (C.c_int, [P, I64P, C.c_int, C.POINTER(GpuSpec), C.POINTER(Weights), C.POINTER(SchedOpts),
                                     C.c_int, C.c_int, I64P, I64P, I64P, I64P]),
    "pmg_pipeline_inlined": (C.c_int, [P, I64P, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "pmg_pipeline_rewritten": (C.c_int, [P, I64P, C.c_int, C.POINTER(SchedOpts), C.c_char_p, C.c_size_t,
                                        C.POINTER(C.c_size_t)]),
    "pmg_run_band": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(Buf), C.c_int, C.POINTER(Buf), C.c_int, C.c_void_p,
                               C.c_void_p]),
    "pmg_band_exchange": (C.c_int, [P, C.c_int, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "pmg_band_exchange_host": (C.c_int, [P, I64P, C.c_int, C.POINTER(GpuSpec), C.POINTER(Weights), C.POINTER(SchedOpts),
                                         C.c_int, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "pmg_run_band_groups": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(Buf), C.c_int, C.POINTER(Buf),
                                      C.c_int, C.c_void_p, C.c_void_p]),
    "pmg_run_host": (C.c_int, [P, C.POINTER(Buf), C.c_int, C.POINTER(Buf), C.c_int, C.POINTER(Buf), C.POINTER(Buf),
                               C.c_void_p, C.c_int, C.c_void_p]),
    "pmg_selftest_shuffle": (C.c_int, [C.c_int, C.POINTER(C.c_int32)]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = sorted(_sig)


def check(status):
    if status != PMG_OK:
        raise PmgError(status, lib.pmg_last_error().decode(errors="replace"))


def call_json(fn, *args):
    need = C.c_size_t(0)
    check(fn(*args, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check(fn(*args, buf, need.value, C.byref(need)))
    return json.loads(buf.value.decode())


def i64arr(vals):
    vals = list(vals)
    return (C.c_int64 * max(1, len(vals)))(*vals), len(vals)

"""Builds paper_1909_07190_b200/libpmg.so (host C++17 + NVRTC; device code is compiled for sm_100a by NVRTC
at plan time from the hand-written csrc/kernels/pmg_otpw.cuh plus the emitted stage bodies).

    python paper_1909_07190_b200/build_lib.py          # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
LIB = HERE / "libpmg.so"
SOURCES = ["parse.cpp", "analysis.cpp", "inline.cpp", "factor.cpp", "phase.cpp", "group.cpp", "emit.cpp", "select.cpp", "runtime.cpp", "capi.cpp",
           "selftest.cpp"]


def embed_header() -> Path:
    src = (CSRC / "kernels" / "pmg_otpw.cuh").read_text()
    if ")PMGHDR\"" in src:
        raise RuntimeError("delimiter clash in pmg_otpw.cuh")
    out = CSRC / "kernels_embed.inc"
    text = f'static const char* kOtpwHeader = R"PMGHDR({src})PMGHDR";\n'
    if not out.exists() or out.read_text() != text:
        out.write_text(text)
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    embed_header()
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.hpp")) + [CSRC / "kernels_embed.inc",
                                                                      HERE.parent / "include" / "pmg.h"]
    if LIB.exists() and not force and all(LIB.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return LIB
    objdir = HERE.parent / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    cflags = ["g++", "-O2", "-g", "-std=c++17", "-fPIC", "-Wall", "-Wno-unused-function", f"-I{CUDA}/include"]
    hdr_time = max(d.stat().st_mtime for d in deps if d.suffix in (".hpp", ".inc", ".h"))

    def compile_one(src: str) -> Path:
        obj = objdir / (src + ".o")
        s = CSRC / src
        if obj.exists() and not force and obj.stat().st_mtime >= max(s.stat().st_mtime, hdr_time):
            return obj
        cmd = cflags + ["-c", str(s), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        return obj

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = ["g++", "-shared", "-o", str(LIB) + ".tmp"] + [str(o) for o in objs]
    cmd += [f"-L{CUDA}/lib64", "-lnvrtc", "-ldl", "-pthread", f"-Wl,-rpath,{CUDA}/lib64",
            "-Wl,--version-script=" + str(CSRC / "exports.map")]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

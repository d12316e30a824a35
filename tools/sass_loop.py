"""Emit + compile one group kernel of a workload (host only, NVRTC) and print the instruction mix of the
interior kernel's main loop (the largest backward-branch body), for quick checks before GPU time.

    python tools/sass_loop.py harris vec=4,chunks=1,rows=112,warps=1,prefetch=4 [group_index]
"""
import collections
import glob
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_07190_b200 as pmg  # noqa: E402
import pmg_inputs as PI  # noqa: E402


def main():
    name = sys.argv[1]
    kv = dict(x.split("=") for x in sys.argv[2].split(",")) if len(sys.argv) > 2 and sys.argv[2] else {}
    gi = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 0
    wl = PI.WORKLOADS[name]
    pipe = pmg.Pipeline(wl.text)
    opts = pmg.sched_opts(**{k: int(v) for k, v in kv.items()}) if kv else None
    rep = pipe.precompile(wl.params, "/tmp/pmg_sass", opts=opts)
    k = rep["kernels"][gi]
    print(k)
    src = pipe.emit(wl.params, opts=opts)["groups"][gi]["source"]
    cub = None
    for f in glob.glob("/tmp/pmg_sass/*.cu") + glob.glob("build/cubin_cache/*.cu"):
        if open(f).read() == src:
            cub = f[:-3] + ".cubin"
    sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
    # keep only the interior kernel's function body
    body, on = [], False
    for line in sass.splitlines():
        if "Function :" in line:
            on = line.strip().endswith(" " + k["name"])
            continue
        if on:
            body.append(line)
    ins = []
    for line in body:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    a2i = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA\s+(0x[0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a and int(m.group(1), 16) in a2i:
            j = a2i[int(m.group(1), 16)]
            body_ = ins[j:i + 1]
            nstg = sum(1 for _, x in body_ if "STG" in x)
            nbra = sum(1 for _, x in body_ if re.search(r"BRA\s+0x", x) and not x.startswith("@"))
            loops.append((i - j, j, i, nstg))
    # the main row loop: the innermost loop that stores rows (fewest instructions among loops with stores)
    # the unrolled main loop: the loop with the most row stores
    _, lo, hi, _ = max(loops, key=lambda l: (l[3], -l[0]))
    c = collections.Counter()
    for a, t in ins[lo:hi + 1]:
        op = t.split()[1] if t.startswith("@") else t.split()[0]
        c[op.split(".")[0]] += 1
    stg = c["STG"] or 1
    print(f"main loop: {hi - lo + 1} instructions, {stg} rows -> {(hi - lo + 1) / stg:.1f} per row")
    fp = sum(v for k_, v in c.items() if k_ in ("FADD", "FMUL", "FFMA", "FADD2", "FMUL2", "FFMA2"))
    print(f"FP {fp / stg:.1f}/row, other {(hi - lo + 1 - fp) / stg:.1f}/row")
    print(", ".join(f"{k_} {v}" for k_, v in c.most_common()))
    if "-v" in sys.argv:
        for a, t in ins[lo:hi + 1]:
            op = t.split()[1] if t.startswith("@") else t.split()[0]
            if not op.startswith(("FADD", "FMUL", "FFMA")):
                print(hex(a), t)


if __name__ == "__main__":
    main()

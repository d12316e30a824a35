"""Summarise ncu output into a committed JSON under profiles/ (DESIGN.md §11).

    python tools/ncu_summary.py --workload harris --round r01 \
        --launches gpurun_out/r1/launches_harris.csv --full gpurun_out/r1/harris_full.ncu-rep

* launches: the `--metrics gpu__time_duration.sum --clock-control none` list of the bench command (cold-cache,
  serialised per-launch times): per-kernel count, mean, share of the GPU time.
* full: one `--set full` capture (the kernels of one pipeline run): time, DRAM bytes, issue/pipe utilisation,
  occupancy, registers, instruction count, top stall reasons.  `dram_bytes_per_launch` (read + write of every
  kernel of one run) is what bench.py reports as `roofline.traffic`.
Writes profiles/ncu_<workload>_<round>.json and refreshes profiles/ncu_<workload>_summary.json."""
import argparse
import csv
import io
import json
import subprocess
from collections import OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

FULL_METRICS = OrderedDict([
    ("time_us", "gpu__time_duration.sum"),
    ("dram_read_bytes", "dram__bytes_read.sum"),
    ("dram_write_bytes", "dram__bytes_write.sum"),
    ("dram_tbps", "dram__bytes.sum.per_second"),
    ("sm_clock_ghz", "sm__cycles_elapsed.avg.per_second"),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("fma_pipe_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("alu_pipe_pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("warp_instructions", "smsp__inst_executed.sum"),
    ("registers_per_thread", "launch__registers_per_thread"),
    ("grid_size", "launch__grid_size"),
    ("block_size", "launch__block_size"),
    ("smem_lsu_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
])
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ns": 1e-3, "ms": 1e3,
              "Tbyte/s": 1, "Gbyte/s": 1e-3, "Ghz": 1, "Mhz": 1e-3}


def fnum(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = fnum(r[vi])
        if v is None:
            continue
        v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}.get(r[ui], 1.0)
        per.setdefault(r[ki], []).append(v)
    total = sum(sum(v) for v in per.values())
    return {"total_gpu_us": total, "kernels": [
        {"name": k, "launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / total if total else None}
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))]}


def full(path):
    if str(path).endswith(".csv"):   # a raw-page CSV exported on the GPU box (ncu -i X.ncu-rep --page raw --csv)
        out = Path(path).read_text()
    else:
        out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    ks = []
    for r in data:
        k = {"name": r[h.index("Kernel Name")]}
        for key, m in FULL_METRICS.items():
            if m not in h:
                k[key] = None
                continue
            i = h.index(m)
            v = fnum(r[i])
            if v is not None and key in ("dram_read_bytes", "dram_write_bytes", "time_us", "dram_tbps", "sm_clock_ghz"):
                v *= UNIT_SCALE.get(units[i], 1)
            k[key] = v
        stalls = {}
        for i, n in enumerate(h):
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                v = fnum(r[i])
                if v:
                    stalls[n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        k["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        ks.append(k)
    return ks


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", required=True)
    ap.add_argument("--round", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    res = {"workload": a.workload, "round": a.round, "note": a.note}
    if a.launches:
        res["launch_list"] = launches(a.launches)
        res["launch_list"]["source"] = ("ncu --metrics gpu__time_duration.sum --clock-control none python bench.py "
                                        "(cold-cache, serialised launches)")
    if a.full:
        ks = full(a.full)
        # the capture holds whole pipeline runs: group kernels by name, keep the first launch of each per run
        seen, run = set(), []
        for k in ks:
            if k["name"] in seen:
                break
            seen.add(k["name"])
            run.append(k)
        res["full"] = {"source": "ncu --set full --clock-control none --import-source on (one pipeline run)",
                       "kernels": run}
        rd = sum(k["dram_read_bytes"] or 0 for k in run)
        wr = sum(k["dram_write_bytes"] or 0 for k in run)
        res["dram_bytes_per_launch"] = rd + wr
        res["dram_bytes_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum summed over the kernels of one "
                                  "pipeline run (interior + border kernels), i.e. per bench step")
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    (prof / f"ncu_{a.workload}_{a.round}.json").write_text(json.dumps(res, indent=1) + "\n")
    (prof / f"ncu_{a.workload}_summary.json").write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()

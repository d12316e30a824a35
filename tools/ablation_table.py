"""Summarise tools/ablation.sh: one row per (workload, variant) with the bench time and the ncu counters."""
import csv
import glob
import json
import os
import sys

d = sys.argv[1]
print(f"{'workload':9s} {'variant':14s} {'us(bench)':>9s} {'us(ncu)':>8s} {'barrier%':>8s} {'membar%':>7s} {'shortsb%':>8s} "
      f"{'longsb%':>7s} {'warps%':>6s} {'regs':>4s} {'gl.ld.sect':>11s} {'smem.bc':>9s} {'inst(M)':>8s} {'issue%':>6s}")
for f in sorted(glob.glob(os.path.join(d, "ncu_*.csv"))):
    wl, var = os.path.basename(f)[4:-4].split("_", 1)
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows:
        continue
    h = rows[0]
    m = {r[h.index("Metric Name")]: r[h.index("Metric Value")] for r in rows[1:]}
    g = lambda k: float(str(m.get(k, "nan")).replace(",", "") or "nan")
    us = float("nan")
    for j in glob.glob(os.path.join(d, f"{wl}-*.json")):
        pass
    bench = [x for x in glob.glob(os.path.join(d, f"{wl}-*.json"))]
    key = {"OTPW_reg": "smem_chunks=0", "OTPW_shared": "smem_chunks=1", "OTPW_shared2": "smem_chunks=2"}
    for b in bench:
        ok = ("PMG_OTPTB" in b) == var.startswith("OTPTB")
        want = "smem_chunks=1" if var.endswith("shared") else "smem_chunks=2" if var.endswith("shared2") else "smem_chunks=0"
        if ok and want in b:
            try:
                us = json.loads(open(b).read().strip().splitlines()[-1])["ms_per_step"] * 1e3
            except Exception:
                pass
    print(f"{wl:9s} {var:14s} {us:9.2f} {g('gpu__time_duration.sum')/1e3:8.2f} "
          f"{g('smsp__warp_issue_stalled_barrier_per_warp_active.pct'):8.2f} {g('smsp__warp_issue_stalled_membar_per_warp_active.pct'):7.2f} "
          f"{g('smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct'):8.2f} {g('smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct'):7.2f} "
          f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} {g('launch__registers_per_thread'):4.0f} "
          f"{g('l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum'):11.0f} "
          f"{g('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum') + g('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum'):9.0f} "
          f"{g('smsp__inst_executed.sum')/1e6:8.2f} {g('smsp__issue_active.avg.pct_of_peak_sustained_active'):6.1f}")

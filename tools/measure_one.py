"""One per-config measurement (bench.measure_config) printed as a compact line: python tools/measure_one.py <workload> [tune]"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

wl = sys.argv[1]
tune = len(sys.argv) > 2 and sys.argv[2] == "tune"
r = bench.measure_config(wl, 0, 20, 5, tune=tune)
env = ",".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("PMG_"))
print(f"{wl:18s} {env:28s} tune={int(tune)} {r['ms_per_run']*1e3:8.2f} us  hbm {r['hbm_frac']:.3f}  alu {r['alu_frac']:.3f}  groups {r['groups']} "
      f"launches {r['launches_per_run']}  plan {r['plan_s']} s  {r['schedule'][:4]}")

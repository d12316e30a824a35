import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import json, paper_1909_07190_b200 as pmg, pmg_inputs as PI
wl=PI.WORKLOADS["harris"]; p=pmg.Pipeline(wl.text)
s=p.schedule(wl.params)
g=s["groups"][0]; print("schedule()", {k:g["config"][k] for k in ["V","TX","TH","NW","PREF","regs_est"]}, g["cost"]["estUs"])
plan=pmg.Plan(p, wl.params)
d=plan.describe(); g=d["schedule"]["groups"][0]; print("plan", {k:g["config"][k] for k in ["V","TX","TH","NW","PREF","regs_est"]}, g["cost"]["estUs"])
q=pmg.query_gpu_spec(0); print({f: getattr(q,f) for f,_ in q._fields_ if f!="name"})
b=pmg.gpu_spec("b200"); print({f: getattr(b,f) for f,_ in b._fields_ if f!="name"})

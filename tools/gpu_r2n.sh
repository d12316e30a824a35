# pair-shared box sums + border-row selection: reassoc / measured-selection parity, then the default bench line
mkdir -p gpurun_out/r2n
( time timeout 900 python -m pytest tests/test_gpu_reassoc.py tests/test_gpu_parity.py -q -x -k "reassoc or measured_selection" --durations=5 ) > gpurun_out/r2n/pytest.txt 2>&1; tail -8 gpurun_out/r2n/pytest.txt
( time timeout 1200 python bench.py ) > gpurun_out/r2n/bench.json 2> gpurun_out/r2n/bench.err
python - <<PY
import json
d = json.loads(open("gpurun_out/r2n/bench.json").read().strip().splitlines()[-1])
print("headline", round(d["ms_per_step"] * 1e3, 2), "us", round(d["roofline"]["hbm"]["frac"], 3), [(c["V"], c["TX"], c["TH"], c["PREF"], c.get("TH_b")) for c in d["config"]["schedule"]], d["clocks"])
for k, v in d["per_config"].items():
    print(k, round(v.get("ms_per_run", 0) * 1e3, 1), v.get("hbm_frac"), v.get("groups"), v.get("launches_per_run"), v.get("schedule"), v.get("error"))
PY
tail -3 gpurun_out/r2n/bench.err

# merged x-edge launches for bands + graph-timed measured selection: parity, band projection, per-config lines
mkdir -p gpurun_out/r2k
( time timeout 900 python -m pytest tests/test_gpu_modes.py tests/test_gpu_fullsize.py tests/test_gpu_exchange.py tests/test_gpu_parity.py -q -x \
   -k "band or exchange or measured_selection" --durations=8 ) > gpurun_out/r2k/pytest.txt 2>&1; tail -14 gpurun_out/r2k/pytest.txt
for n in 2 4 8; do
  timeout 600 python bench.py --simulate-bands $n --no-cpu-baseline --no-per-config --no-e2e > gpurun_out/r2k/harris_b$n.json 2> gpurun_out/r2k/harris_b$n.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2k/harris_b$n.json').read().strip().splitlines()[-1]); print('bands $n', round(d['ms_per_step']*1e3,2), 'us', [(c['V'],c['TX'],c['TH'],c['PREF']) for c in d['config']['schedule']], d['gpu_launches']//d['steps'], 'launches')"
done
( time timeout 1200 python bench.py ) > gpurun_out/r2k/bench.json 2> gpurun_out/r2k/bench.err
python - <<PY
import json
d = json.loads(open("gpurun_out/r2k/bench.json").read().strip().splitlines()[-1])
print("headline", round(d["ms_per_step"] * 1e3, 2), "us", round(d["roofline"]["hbm"]["frac"], 3), [(c["V"], c["TX"], c["TH"], c["PREF"]) for c in d["config"]["schedule"]])
for k, v in d["per_config"].items():
    print(k, round(v.get("ms_per_run", 0) * 1e3, 1), v.get("groups"), v.get("launches_per_run"), v.get("schedule"), v.get("error"))
PY
tail -3 gpurun_out/r2k/bench.err

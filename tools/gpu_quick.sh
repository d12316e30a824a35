# quick GPU iteration: selected tests, then the Harris bench in both arithmetic modes (no per-config lines)
# usage: bash tools/gpu_quick.sh <tag> [pytest files...]
tag=${1:-r}; shift
mkdir -p gpurun_out/$tag
if [ $# -gt 0 ]; then
  ( time timeout 900 python -m pytest "$@" -q -x --durations=15 ) > gpurun_out/$tag/pytest.txt 2>&1; tail -25 gpurun_out/$tag/pytest.txt
fi
timeout 600 python bench.py --no-per-config --no-cpu-baseline --no-e2e > gpurun_out/$tag/bench_reassoc.json 2> gpurun_out/$tag/bench_reassoc.err
timeout 600 python bench.py --no-per-config --no-cpu-baseline --no-e2e --exact > gpurun_out/$tag/bench_exact.json 2> gpurun_out/$tag/bench_exact.err
for f in reassoc exact; do python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/$tag/bench_$f.json").read().strip().splitlines()[-1])
    print("$f", round(d["ms_per_step"] * 1e3, 2), "us", "hbm", round(d["roofline"]["hbm"]["frac"], 3), d["roofline"]["bound"],
          round(d["roofline"]["frac"], 3), [ (k["name"], k["regs"]) for k in d["config"]["kernels"]], d["config"]["launch"])
except Exception as e:
    print("$f failed", e); print(open("gpurun_out/$tag/bench_$f.err").read()[-2000:])
PY
done

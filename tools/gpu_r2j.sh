# camera with hoisted colour-matrix loads (parity + timings); unsharp configuration check
mkdir -p gpurun_out/r2j
( time timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_guards.py -q -x -k "camera" ) > gpurun_out/r2j/pytest.txt 2>&1; tail -4 gpurun_out/r2j/pytest.txt
timeout 900 python - <<PY
import sys
sys.path.insert(0, ".")
import bench
for tune in (False, True):
    r = bench.measure_config("camera", 0, 20, 5, tune=tune)
    print("camera tune", tune, round(r["ms_per_run"] * 1e3, 1), r["groups"], r["launches_per_run"], r["schedule"], flush=True)
PY
for v in ";vec=1,chunks=4,rows=24,warps=1,prefetch=4" ";vec=4,chunks=1,rows=48,warps=1,prefetch=4" ";vec=4,chunks=1,rows=32,warps=1,prefetch=4" \
         "PMG_PDL=0;vec=1,chunks=4,rows=24,warps=1,prefetch=4" ";vec=2,chunks=2,rows=24,warps=1,prefetch=4" ";vec=4,chunks=1,rows=24,warps=1,prefetch=6"; do
  bash tools/bench_variants.sh r2j unsharp "$v"
done
timeout 300 python bench.py --workload unsharp --exact --no-cpu-baseline --no-per-config --no-e2e --opts vec=1,chunks=4,rows=24,warps=1,prefetch=4 > gpurun_out/r2j/u_exact.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r2j/u_exact.json').read().strip().splitlines()[-1]); print('unsharp exact V1TX4TH24', round(d['ms_per_step']*1e3,2))"

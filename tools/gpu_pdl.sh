# PDL A/B: parity subset with PDL on, then the per-config lines (model schedules) with PMG_PDL=0 and 1
mkdir -p gpurun_out/r2f
( time timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exchange.py -q -x -k "local_laplacian or pyramid or camera_parity or multiscale or ll_small or harris" ) > gpurun_out/r2f/pytest.txt 2>&1; tail -4 gpurun_out/r2f/pytest.txt
for pdl in 0 1; do
  PMG_PDL=$pdl timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-tune --opts vec=4,chunks=1,rows=62,warps=1,prefetch=6 > gpurun_out/r2f/bench_pdl$pdl.json 2> gpurun_out/r2f/bench_pdl$pdl.err
  PMG_PDL=$pdl timeout 900 python - <<PY
import json, sys
sys.path.insert(0, ".")
import bench
out = {}
for n in ["unsharp", "camera", "local_laplacian", "pyramid_blend", "multiscale_interp", "blur"]:
    try:
        r = bench.measure_config(n, 0, 20, 5, tune=False)
        out[n] = (round(r["ms_per_run"] * 1e3, 1), r["groups"], r["launches_per_run"])
    except Exception as e:
        out[n] = str(e)[:200]
print("PDL=$pdl", out)
PY
done
python -c "
import json
for p in (0, 1):
    d = json.loads(open(f'gpurun_out/r2f/bench_pdl{p}.json').read().strip().splitlines()[-1]); print('harris PDL', p, round(d['ms_per_step']*1e3, 2))"

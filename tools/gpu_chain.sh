# chains + down-sampling clones: parity subset, then per-config model-schedule timings for each switch setting
mkdir -p gpurun_out/r2g
( time timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_exchange.py -q -x --durations=12 \
   -k "local_laplacian or pyramid or multiscale or camera_parity or whole_image or ll_small" ) > gpurun_out/r2g/pytest.txt 2>&1; tail -18 gpurun_out/r2g/pytest.txt
for cfg in "PMG_CHAIN=0 PMG_DOWN_CLONE=0" "PMG_CHAIN=1 PMG_DOWN_CLONE=0" "PMG_CHAIN=0 PMG_DOWN_CLONE=1" "PMG_CHAIN=1 PMG_DOWN_CLONE=1"; do
  env $cfg timeout 900 python - <<PY
import json, sys
sys.path.insert(0, ".")
import bench
out = {}
for n in ["local_laplacian", "pyramid_blend", "multiscale_interp", "camera"]:
    try:
        r = bench.measure_config(n, 0, 20, 5, tune=False)
        out[n] = (round(r["ms_per_run"] * 1e3, 1), r["groups"], r["launches_per_run"])
    except Exception as e:
        out[n] = str(e)[:300]
print("$cfg", out, flush=True)
PY
done
timeout 900 python - <<PY
import sys
sys.path.insert(0, ".")
import bench
for n in ["local_laplacian", "pyramid_blend", "multiscale_interp"]:
    r = bench.measure_config(n, 0, 20, 5, tune=True)
    print("tuned", n, round(r["ms_per_run"] * 1e3, 1), r["groups"], r["launches_per_run"], flush=True)
PY

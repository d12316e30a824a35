# border-tile height for the pyramids' small levels: per-config model-schedule times for PMG_BORDER_TH = 8 (default), 4, 2
mkdir -p gpurun_out/r2m
for th in 8 4 2 16; do
  PMG_BORDER_TH=$th timeout 900 python - <<PY
import sys
sys.path.insert(0, ".")
import bench
out = {}
for n in ["local_laplacian", "pyramid_blend", "multiscale_interp", "camera"]:
    try:
        r = bench.measure_config(n, 0, 20, 5, tune=False)
        out[n] = round(r["ms_per_run"] * 1e3, 1)
    except Exception as e:
        out[n] = str(e)[:200]
print("BORDER_TH=$th", out, flush=True)
PY
done

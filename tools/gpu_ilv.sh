mkdir -p gpurun_out/r2s
( time timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_modes.py tests/test_gpu_guards.py -q -x -k "camera" --durations=5 ) > gpurun_out/r2s/pytest.txt 2>&1; tail -12 gpurun_out/r2s/pytest.txt
timeout 600 python - <<PY
import sys
sys.path.insert(0, ".")
import bench
r = bench.measure_config("camera", 0, 20, 5, tune=True)
print("camera cached", round(r["ms_per_run"] * 1e3, 1), r["groups"], r["launches_per_run"])
PY
PMG_ILV=0 timeout 600 python - <<PY
import sys
sys.path.insert(0, ".")
import bench
r = bench.measure_config("camera", 0, 20, 5, tune=True)
print("camera cached, no interleave fusion", round(r["ms_per_run"] * 1e3, 1), r["groups"], r["launches_per_run"])
PY

mkdir -p gpurun_out/r2l
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "camera" > gpurun_out/r2l/pytest.txt 2>&1; tail -3 gpurun_out/r2l/pytest.txt
for wl in camera local_laplacian multiscale_interp pyramid_blend unsharp; do
  for sc in 0 1; do PMG_SCALED=$sc timeout 600 python tools/measure_one.py $wl 2>&1 | tail -1; done
done
timeout 900 python tools/measure_one.py camera tune 2>&1 | tail -1
PMG_UP_SPLIT=0 timeout 600 python tools/measure_one.py camera 2>&1 | tail -1
PMG_PHASE_SPLIT=0 timeout 600 python tools/measure_one.py local_laplacian 2>&1 | tail -1

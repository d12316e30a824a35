mkdir -p gpurun_out/r2b
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -x -k "harris or unsharp or blur or operator or camera_parity" > gpurun_out/r2b/pytest.txt 2>&1; tail -3 gpurun_out/r2b/pytest.txt
bash tools/bench_variants.sh r2b harris ";" "PMG_FENCE=1;" "PMG_XEDGE=0;" \
  ";vec=4,chunks=1,rows=96,warps=1,prefetch=4" ";vec=4,chunks=1,rows=96,warps=1,prefetch=4,regcap=80" \
  ";vec=4,chunks=1,rows=104,warps=1,prefetch=4,regcap=80" ";vec=4,chunks=1,rows=112,warps=1,prefetch=4,regcap=80" \
  ";vec=4,chunks=1,rows=128,warps=1,prefetch=4,regcap=80" "PMG_FENCE=1;vec=4,chunks=1,rows=104,warps=1,prefetch=4" \
  "PMG_XEDGE=0;vec=4,chunks=1,rows=96,warps=1,prefetch=4,regcap=80"
bash tools/bench_variants.sh r2b unsharp ";" "PMG_XEDGE=0;"

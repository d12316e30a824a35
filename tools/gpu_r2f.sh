timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -q -x -k "harris or unsharp or blur or operator or camera_parity or band" > gpurun_out/r2f/pytest.txt 2>&1; tail -3 gpurun_out/r2f/pytest.txt
bash tools/bench_variants.sh r2f harris ";" ";vec=4,chunks=1,rows=100,warps=1,prefetch=4" ";vec=4,chunks=2,rows=80,warps=1,prefetch=4" ";vec=4,chunks=1,rows=96,warps=1,prefetch=4" \
   ";vec=4,chunks=2,rows=48,warps=1,prefetch=4" ";vec=2,chunks=2,rows=100,warps=1,prefetch=4" ";vec=4,chunks=1,rows=100,warps=1,prefetch=2" ";vec=4,chunks=1,rows=100,warps=1,prefetch=6"
bash tools/bench_variants.sh r2f unsharp ";" ";vec=4,chunks=1,rows=48,warps=1,prefetch=4" ";vec=4,chunks=1,rows=24,warps=1,prefetch=4" ";vec=2,chunks=2,rows=24,warps=1,prefetch=4"
bash tools/bench_variants.sh r2f camera ";"
bash tools/bench_variants.sh r2f local_laplacian ";"

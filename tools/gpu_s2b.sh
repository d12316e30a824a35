# V=8 lanes for Harris / unsharp; per-kernel launch lists of camera and local Laplacian
tag=s2b
mkdir -p gpurun_out/$tag
python tools/sweep.py harris vec=4,chunks=1,rows=96,warps=1,prefetch=4 vec=8,chunks=1,rows=96,warps=1,prefetch=4 vec=8,chunks=1,rows=64,warps=1,prefetch=4 vec=8,chunks=1,rows=48,warps=1,prefetch=4 vec=8,chunks=1,rows=128,warps=1,prefetch=4 vec=8,chunks=1,rows=96,warps=1,prefetch=2 vec=8,chunks=1,rows=96,warps=1,prefetch=3 > gpurun_out/$tag/harris_v8.txt 2>&1
python tools/sweep.py unsharp vec=1,chunks=4,rows=24,warps=1,prefetch=4 vec=8,chunks=1,rows=24,warps=1,prefetch=4 vec=8,chunks=1,rows=32,warps=1,prefetch=4 vec=4,chunks=2,rows=24,warps=1,prefetch=4 > gpurun_out/$tag/unsharp_v8.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches_camera.csv python tools/run_once.py camera auto 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches_ll.csv python tools/run_once.py local_laplacian auto 2 > /dev/null 2>&1
cat gpurun_out/$tag/*.txt

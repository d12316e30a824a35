# scaled streams: parity (new scaled-stream tests, camera, LL), then timings
tag=s2e
mkdir -p gpurun_out/$tag
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "scaled or camera or local or harris_parity or unsharp" > gpurun_out/$tag/pytest_parity.txt 2>&1; tail -15 gpurun_out/$tag/pytest_parity.txt
for w in camera local_laplacian; do timeout 300 python tools/sweep.py $w > gpurun_out/$tag/auto_$w.txt 2>&1; PMG_SCALED=0 timeout 300 python tools/sweep.py $w > gpurun_out/$tag/noscale_$w.txt 2>&1; done
GOS=0.1.1.1.1.1.1.1.1.1.1.1.1.2.2.2.2.2
timeout 300 python tools/sweep.py camera gos=$GOS,vec=2 gos=$GOS,vec=4 gos=$GOS,vec=4,chunks=1 gos=$GOS,vec=2,chunks=2 > gpurun_out/$tag/camera_gos.txt 2>&1
head -30 gpurun_out/$tag/*.txt

# camera groupings (broadcast fusion, scaled-stream cap), c_gather settings; PREF depth for unsharp / Harris
tag=s2g
mkdir -p gpurun_out/$tag
F=0.1.1.1.1.1.1.1.1.1.1.1.1.2.2.2.2.2
S=0.1.1.1.1.1.1.1.1.1.1.1.1.2.3.4.5.5
for cg in 12 6 3; do PMG_TM=10,2,0,1800,1,3,4,$cg timeout 300 python tools/sweep.py camera > gpurun_out/$tag/camera_cg$cg.txt 2>&1; done
timeout 600 python tools/sweep.py camera gos=$F,vec=4,chunks=1,rows=8 gos=$F,vec=4,chunks=1,rows=16 gos=$F,vec=2,chunks=2,rows=8 gos=$F,vec=4,chunks=2,rows=8 gos=$S,vec=4,chunks=1,rows=8 > gpurun_out/$tag/camera_gos.txt 2>&1
timeout 300 python tools/sweep.py unsharp vec=2,chunks=2,rows=24,warps=1,prefetch=4 vec=2,chunks=2,rows=24,warps=1,prefetch=6 vec=2,chunks=2,rows=24,warps=1,prefetch=8 vec=1,chunks=4,rows=24,warps=1,prefetch=8 vec=4,chunks=1,rows=24,warps=1,prefetch=8 > gpurun_out/$tag/unsharp_pref.txt 2>&1
timeout 300 python tools/sweep.py harris vec=4,chunks=1,rows=96,warps=1,prefetch=4 vec=4,chunks=1,rows=96,warps=1,prefetch=6 vec=4,chunks=1,rows=96,warps=1,prefetch=8 > gpurun_out/$tag/harris_pref.txt 2>&1
timeout 300 python tools/sweep.py local_laplacian > gpurun_out/$tag/ll.txt 2>&1
for f in gpurun_out/$tag/*.txt; do echo $f; cat $f; done

# Harris: taller warp tiles (less y-overlap recompute) than the selector's 96-row maximum
tag=s2q
mkdir -p gpurun_out/$tag
G=gos=0.0.0.0.0.0.0.0.0.0.0
timeout 900 python tools/sweep.py harris $G,vec=4,chunks=1,rows=96,warps=1,prefetch=4 $G,vec=4,chunks=1,rows=128,warps=1,prefetch=4 $G,vec=4,chunks=1,rows=160,warps=1,prefetch=4 $G,vec=4,chunks=1,rows=192,warps=1,prefetch=4 $G,vec=4,chunks=1,rows=112,warps=1,prefetch=4 $G,vec=4,chunks=1,rows=144,warps=1,prefetch=4 > gpurun_out/$tag/harris_th.txt 2>&1
cat gpurun_out/$tag/harris_th.txt

# x-border tiles in the interior kernel (PMG_XIN) on/off; camera broadcast fusion (R,G,B into corrected/curved)
tag=s2d
mkdir -p gpurun_out/$tag
for xin in 0 1; do
  for w in harris unsharp blur camera; do PMG_XIN=$xin timeout 300 python tools/sweep.py $w > gpurun_out/$tag/xin${xin}_$w.txt 2>&1; done
done
GOS=0.1.1.1.1.1.1.1.1.1.1.1.1.2.2.2.2.2
PMG_XIN=0 timeout 300 python tools/sweep.py camera gos=$GOS gos=$GOS,vec=2 gos=$GOS,vec=4 gos=0.1.1.1.1.1.1.1.1.1.1.1.1.2.2.2.3.3 > gpurun_out/$tag/camera_gos.txt 2>&1
head -50 gpurun_out/$tag/*.txt

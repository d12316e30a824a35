# x-border kernel (PMG_XK = rows per x-border tile; 0 = off): parity of everything, then timings
tag=s2f
mkdir -p gpurun_out/$tag
for xk in 0 24 16 32 48; do
  for w in harris unsharp; do PMG_XK=$xk timeout 300 python tools/sweep.py $w > gpurun_out/$tag/xk${xk}_$w.txt 2>&1; done
done
for xk in 0 24; do for w in camera local_laplacian blur; do PMG_XK=$xk timeout 300 python tools/sweep.py $w > gpurun_out/$tag/xk${xk}_$w.txt 2>&1; done; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$tag/pytest_gpu.txt 2>&1; tail -15 gpurun_out/$tag/pytest_gpu.txt
for f in gpurun_out/$tag/xk*.txt; do echo $f; cat $f; done

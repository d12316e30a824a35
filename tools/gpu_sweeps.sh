# schedule sweeps for the time-model fit: bash tools/gpu_sweeps.sh <tag>
tag=${1:-r}
mkdir -p gpurun_out/$tag
for w in harris unsharp blur camera; do timeout 1200 python tools/sweep.py $w grid > gpurun_out/$tag/sweep_$w.txt 2>&1; done
tail -n 2 gpurun_out/$tag/*.txt

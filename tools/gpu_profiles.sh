# ncu evidence for profiles/ (B200_PROFILING.md recipe): launch list of the bench's timed configuration and one
# --set full capture per workload.  bash tools/gpu_profiles.sh <tag> "<harris opts>"
tag=${1:-prof}; HO=${2:-vec=4,chunks=1,rows=100,warps=1,prefetch=4}
mkdir -p gpurun_out/$tag
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread --clock-control none --csv \
  --log-file gpurun_out/$tag/launches_harris.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-graph --no-e2e \
  --no-per-config --opts $HO > gpurun_out/$tag/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pmg_g0 -c 3 -o gpurun_out/$tag/harris_full \
  python tools/run_once.py harris "$HO" 1 > gpurun_out/$tag/ncu_harris.log 2>&1
for wl in unsharp camera local_laplacian multiscale_interp; do
  timeout 1200 ncu --set full --clock-control none -c 60 -o gpurun_out/$tag/${wl}_full python tools/run_once.py $wl auto 1 \
    > gpurun_out/$tag/ncu_$wl.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/$tag/launches_$wl.csv \
    python tools/run_once.py $wl auto 3 > /dev/null 2>&1
done
# keep the raw-page CSV of every capture (small); the .ncu-rep files themselves stay on the box except Harris's
for f in gpurun_out/$tag/*_full.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null
  case $f in *harris_full*) ;; *) rm -f $f ;; esac
done
ls -la gpurun_out/$tag/

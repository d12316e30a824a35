# ncu evidence for profiles/ (B200_PROFILING.md recipe) of the bench's timed configurations (the cached measured
# selection): per workload a launch list (3 runs) and one --set full capture of one run, exported as the raw-page
# CSV (the .ncu-rep of the pyramids is tens of MB: only Harris's is kept).   bash tools/gpu_profiles.sh <tag>
tag=${1:-prof}
mkdir -p gpurun_out/$tag
for wl in harris unsharp camera local_laplacian; do
  timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread --clock-control none --csv \
    --log-file gpurun_out/$tag/launches_$wl.csv python tools/run_once.py $wl cached 3 > gpurun_out/$tag/run_$wl.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pmg_g -c 40 -o gpurun_out/$tag/${wl}_full \
    python tools/run_once.py $wl cached 1 > gpurun_out/$tag/ncu_$wl.log 2>&1
  ncu -i gpurun_out/$tag/${wl}_full.ncu-rep --page raw --csv > gpurun_out/$tag/${wl}_full_raw.csv 2>/dev/null
  [ "$wl" = harris ] || rm -f gpurun_out/$tag/${wl}_full.ncu-rep
  tail -1 gpurun_out/$tag/ncu_$wl.log
done
du -sh gpurun_out/$tag

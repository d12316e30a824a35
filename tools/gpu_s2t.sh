# N=8 band kernel times (serialised launch list) for the band-scaling analysis
tag=s2t
mkdir -p gpurun_out/$tag
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none --csv --log-file gpurun_out/$tag/launches_band8.csv python bench.py --simulate-bands 8 --steps 3 --warmup 3 --no-graph --no-cpu-baseline > gpurun_out/$tag/band8.log 2>&1
tail -2 gpurun_out/$tag/band8.log

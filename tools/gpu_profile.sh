# ncu launch list + one --set full capture of the bench workload, then the bench line: bash tools/gpu_profile.sh <tag>
tag=${1:-r}
mkdir -p gpurun_out/$tag
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches_harris.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/$tag/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pmg_g0 -c 2 -o gpurun_out/$tag/harris_full python tools/run_once.py harris auto 2 > gpurun_out/$tag/ncu_full.log 2>&1
timeout 600 python bench.py > gpurun_out/$tag/bench.json 2> gpurun_out/$tag/bench.err
tail -c 400 gpurun_out/$tag/bench.json

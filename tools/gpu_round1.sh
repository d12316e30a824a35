set -x
mkdir -p gpurun_out/r1
for w in harris unsharp blur camera; do timeout 900 python tools/sweep.py $w grid > gpurun_out/r1/sweep_$w.txt 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1/launches_harris.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pmg_g0 -c 2 -o gpurun_out/r1/harris_full python tools/run_once.py harris auto 2 > gpurun_out/r1/ncu_full.log 2>&1
timeout 600 python bench.py > gpurun_out/r1/bench.json 2> gpurun_out/r1/bench.err
tail -c 1500 gpurun_out/r1/bench.json

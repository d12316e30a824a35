# Harris (reassociation mode) tile / ring-depth sweep, the bench's launch list and one --set full capture
v=""
for th in 48 64 96 128; do for pf in 4 6 8; do v="$v ;vec=4,chunks=1,rows=$th,warps=1,prefetch=$pf"; done; done
bash tools/bench_variants.sh r2c harris $v ";vec=2,chunks=2,rows=64,warps=1,prefetch=6" ";vec=8,chunks=1,rows=64,warps=1,prefetch=4" ";vec=4,chunks=2,rows=64,warps=1,prefetch=4"
mkdir -p gpurun_out/r2c
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c/launches_harris.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-per-config --no-e2e --no-graph > gpurun_out/r2c/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pmg_g0 -c 3 -o gpurun_out/r2c/harris_full python tools/run_once.py harris vec=4,chunks=1,rows=64,warps=1,prefetch=4,reassoc=1 1 > gpurun_out/r2c/ncu_full.log 2>&1
tail -3 gpurun_out/r2c/ncu_full.log

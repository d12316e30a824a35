mkdir -p gpurun_out/r2e
( time timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_guards.py -q -x --durations=10 ) > gpurun_out/r2e/pytest.txt 2>&1; tail -16 gpurun_out/r2e/pytest.txt
v=""
for o in "rows=62,prefetch=6" "rows=68,prefetch=6" "rows=92,prefetch=6" "rows=60,prefetch=8" "rows=68,prefetch=8" "rows=92,prefetch=8" "rows=124,prefetch=8" "rows=64,prefetch=6" "rows=128,prefetch=6"; do v="$v ;vec=4,chunks=1,warps=1,$o"; done
bash tools/bench_variants.sh r2e harris $v
timeout 600 python bench.py --simulate-bands 8 --exchange --workload local_laplacian --no-cpu-baseline --no-per-config --no-e2e --no-tune > gpurun_out/r2e/ll_x8.json 2> gpurun_out/r2e/ll_x8.err; tail -c 700 gpurun_out/r2e/ll_x8.json; tail -3 gpurun_out/r2e/ll_x8.err
timeout 600 python bench.py --simulate-bands 8 --workload local_laplacian --no-cpu-baseline --no-per-config --no-e2e --no-tune > gpurun_out/r2e/ll_r8.json 2> gpurun_out/r2e/ll_r8.err; tail -c 300 gpurun_out/r2e/ll_r8.json
timeout 600 python bench.py --workload local_laplacian --no-cpu-baseline --no-per-config --no-e2e --no-tune > gpurun_out/r2e/ll_1.json 2> gpurun_out/r2e/ll_1.err; tail -c 300 gpurun_out/r2e/ll_1.json

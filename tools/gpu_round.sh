# one GPU session: parity + auto-vs-best sweeps + ncu launch list / full capture of the bench workload + bench
# usage: bash tools/gpu_round.sh <tag>
set -x
tag=${1:-r}
mkdir -p gpurun_out/$tag
python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -x -q > gpurun_out/$tag/pytest_gpu.txt 2>&1; tail -2 gpurun_out/$tag/pytest_gpu.txt
python tools/sweep.py harris vec=4,chunks=1,rows=32,warps=1,prefetch=4 > gpurun_out/$tag/auto_harris.txt 2>&1
python tools/sweep.py unsharp vec=4,chunks=1,rows=32,warps=1,prefetch=4 vec=2,chunks=2,rows=24,warps=1,prefetch=4 > gpurun_out/$tag/auto_unsharp.txt 2>&1
python tools/sweep.py camera vec=4,chunks=1,rows=16,warps=1,prefetch=4 > gpurun_out/$tag/auto_camera.txt 2>&1
python tools/sweep.py blur > gpurun_out/$tag/auto_blur.txt 2>&1
python tools/sweep.py local_laplacian > gpurun_out/$tag/auto_ll.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches_harris.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$tag/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pmg_g0 -c 2 -o gpurun_out/$tag/harris_full python tools/run_once.py harris auto 2 > gpurun_out/$tag/ncu_full.log 2>&1
timeout 600 python bench.py > gpurun_out/$tag/bench.json 2> gpurun_out/$tag/bench.err
cat gpurun_out/$tag/auto_*.txt
tail -c 600 gpurun_out/$tag/bench.json

# one GPU session: the -m gpu suite (durations), smoke, the default bench line (per-config lines included),
# register-cap variants of the Harris kernel, the launch list of the bench's timed configuration (no measured
# selection under ncu: only the timed kernels appear) and one --set full capture of the Harris kernel.
# usage: bash tools/gpu_round.sh <tag> [harris opts]
tag=${1:-r}; hopts=${2:-vec=4,chunks=1,rows=64,warps=1,prefetch=6}
mkdir -p gpurun_out/$tag
( time timeout 1150 python -m pytest tests -m gpu -q -x --durations=30 ) > gpurun_out/$tag/pytest_gpu.txt 2>&1
tail -42 gpurun_out/$tag/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$tag/smoke.txt 2>&1; tail -3 gpurun_out/$tag/smoke.txt
( time timeout 900 python bench.py ) > gpurun_out/$tag/bench.json 2> gpurun_out/$tag/bench.err
tail -c 1500 gpurun_out/$tag/bench.json; tail -4 gpurun_out/$tag/bench.err
bash tools/bench_variants.sh $tag harris "PMG_CAP_I=80;$hopts" "PMG_CAP_I=72;$hopts" ";$hopts"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches_harris.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-per-config --no-e2e --no-graph --no-tune --opts $hopts > gpurun_out/$tag/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pmg_g0 -c 3 -o gpurun_out/$tag/harris_full \
  python tools/run_once.py harris $hopts,reassoc=1 1 > gpurun_out/$tag/ncu_full.log 2>&1
tail -2 gpurun_out/$tag/ncu_full.log

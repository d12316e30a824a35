# one GPU session: the full -m gpu suite with durations, smoke, then the default bench line
# usage: bash tools/gpu_check.sh <tag>
tag=${1:-r}
mkdir -p gpurun_out/$tag
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$tag/smi.txt 2>&1
( time timeout 1500 python -m pytest tests -m gpu -q -x --durations=40 ) > gpurun_out/$tag/pytest_gpu.txt 2>&1
tail -50 gpurun_out/$tag/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$tag/smoke.txt 2>&1; cat gpurun_out/$tag/smoke.txt | tail -3
( time timeout 900 python bench.py ) > gpurun_out/$tag/bench.json 2> gpurun_out/$tag/bench.err
tail -c 3000 gpurun_out/$tag/bench.json; tail -5 gpurun_out/$tag/bench.err

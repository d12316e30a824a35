# GPU test suite with per-test durations: bash tools/gpu_tests.sh <tag> [pytest args]
tag=${1:-r}; shift
mkdir -p gpurun_out/$tag
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$tag/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=60 "$@" > gpurun_out/$tag/pytest_gpu.txt 2>&1
tail -75 gpurun_out/$tag/pytest_gpu.txt

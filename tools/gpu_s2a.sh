tag=s2a
mkdir -p gpurun_out/$tag
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$tag/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$tag/pytest_gpu.txt 2>&1; tail -3 gpurun_out/$tag/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$tag/smoke.txt 2>&1; tail -2 gpurun_out/$tag/smoke.txt
bash tools/gpu_profile.sh $tag
for w in unsharp camera local_laplacian blur; do timeout 300 python tools/sweep.py $w > gpurun_out/$tag/once_$w.txt 2>&1; tail -3 gpurun_out/$tag/once_$w.txt; done

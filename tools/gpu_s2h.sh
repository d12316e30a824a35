# end-of-session check: full GPU suite, smoke, auto timings of every workload, ncu launch list + full capture, bench
tag=s2h
mkdir -p gpurun_out/$tag
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$tag/pytest_gpu.txt 2>&1; tail -3 gpurun_out/$tag/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$tag/smoke.txt 2>&1; tail -2 gpurun_out/$tag/smoke.txt
for w in harris unsharp camera local_laplacian blur; do timeout 300 python tools/sweep.py $w > gpurun_out/$tag/auto_$w.txt 2>&1; done
bash tools/gpu_profile.sh $tag
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches_camera.csv python tools/run_once.py camera auto 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches_ll.csv python tools/run_once.py local_laplacian auto 2 > /dev/null 2>&1
cat gpurun_out/$tag/auto_*.txt

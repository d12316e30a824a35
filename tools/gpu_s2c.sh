# parity-folding check: camera / LL parity + timings + one ncu --set full of the camera pipe
tag=s2c
mkdir -p gpurun_out/$tag
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/$tag/pytest_parity.txt 2>&1; tail -3 gpurun_out/$tag/pytest_parity.txt
for w in camera local_laplacian harris unsharp; do timeout 300 python tools/sweep.py $w > gpurun_out/$tag/auto_$w.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches_camera.csv python tools/run_once.py camera auto 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pmg_g -c 8 -o gpurun_out/$tag/camera_full python tools/run_once.py camera auto 1 > gpurun_out/$tag/ncu_full.log 2>&1
cat gpurun_out/$tag/auto_*.txt

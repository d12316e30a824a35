# pyramid blend parity + timing; every pipeline at the paper's Table 2 sizes (context for Table 3's V100 times)
tag=s2i
mkdir -p gpurun_out/$tag
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "pyramid" > gpurun_out/$tag/pytest_pb.txt 2>&1; tail -3 gpurun_out/$tag/pytest_pb.txt
timeout 300 python tools/sweep.py pyramid_blend > gpurun_out/$tag/auto_pb.txt 2>&1
PMG_SCALED=0 timeout 300 python tools/sweep.py pyramid_blend > gpurun_out/$tag/noscale_pb.txt 2>&1
timeout 300 python tools/sweep.py harris W=4256x2832 > gpurun_out/$tag/paper_harris.txt 2>&1
timeout 300 python tools/sweep.py unsharp W=4256x2832 > gpurun_out/$tag/paper_unsharp.txt 2>&1
timeout 300 python tools/sweep.py camera W=2592x1968 > gpurun_out/$tag/paper_camera.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches_pb.csv python tools/run_once.py pyramid_blend auto 2 > /dev/null 2>&1
for f in gpurun_out/$tag/*.txt; do echo $f; cat $f; done

# defaults after the scaled-stream opt-in and the select-aware time model: parity of the touched tests, timings
tag=s2j
mkdir -p gpurun_out/$tag
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "scaled or camera or pyramid" > gpurun_out/$tag/pytest.txt 2>&1; tail -3 gpurun_out/$tag/pytest.txt
for w in camera local_laplacian pyramid_blend harris unsharp; do timeout 300 python tools/sweep.py $w > gpurun_out/$tag/auto_$w.txt 2>&1; done
for f in gpurun_out/$tag/auto*.txt; do echo $f; cat $f; done

# measured selection with the best-of-3 statistic: parity + tuned timings
tag=s2p
mkdir -p gpurun_out/$tag
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "measured_selection" > gpurun_out/$tag/pytest.txt 2>&1; tail -3 gpurun_out/$tag/pytest.txt
for w in unsharp camera blur; do timeout 900 python tools/sweep.py $w tune=1 > gpurun_out/$tag/tune_$w.txt 2>&1; done
for f in gpurun_out/$tag/*.txt; do echo $f; cat $f; done

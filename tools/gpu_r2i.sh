mkdir -p gpurun_out/r2i
timeout 1200 python -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "sanitizer or multiscale" --durations=10 > gpurun_out/r2i/pytest.txt 2>&1; tail -15 gpurun_out/r2i/pytest.txt
O="vec=4,chunks=1,rows=100,warps=1,prefetch=4"
for i in 1 2; do bash tools/bench_variants.sh r2i harris ";$O" "PMG_TUNE_GRID=1;"; done
for n in 2 4 8; do timeout 600 python bench.py --simulate-bands $n --no-cpu-baseline --no-per-config > gpurun_out/r2i/bands$n.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r2i/bands$n.json').read().strip().splitlines()[-1]); print('bands $n', d['ms_per_step']*1e3, 'us', [ (c['V'],c['TX'],c['TH']) for c in d['config']['schedule']])"; done

# Harris N = 8 band configurations (simulated on one GPU), then the full -m gpu suite and smoke
mkdir -p gpurun_out/r2i
for o in "vec=4,chunks=1,rows=16,warps=1,prefetch=4" "vec=4,chunks=1,rows=12,warps=1,prefetch=8" "vec=4,chunks=1,rows=16,warps=1,prefetch=6" \
         "vec=4,chunks=1,rows=8,warps=1,prefetch=4" "vec=4,chunks=1,rows=24,warps=1,prefetch=6" "vec=2,chunks=1,rows=16,warps=1,prefetch=4" \
         "vec=2,chunks=1,rows=32,warps=1,prefetch=6" "vec=4,chunks=1,rows=20,warps=1,prefetch=8" "vec=1,chunks=4,rows=16,warps=1,prefetch=4"; do
  timeout 300 python bench.py --simulate-bands 8 --no-cpu-baseline --no-per-config --no-e2e --opts $o > gpurun_out/r2i/b.json 2> gpurun_out/r2i/b.err
  python -c "
import json
try:
    d=json.loads(open('gpurun_out/r2i/b.json').read().strip().splitlines()[-1]); print('bands 8 $o', round(d['ms_per_step']*1e3,2), 'us', d['config']['launch'][:40])
except Exception as e: print('$o failed', open('gpurun_out/r2i/b.err').read()[-300:])"
done
( time timeout 1150 python -m pytest tests -m gpu -q -x --durations=25 ) > gpurun_out/r2i/pytest_gpu.txt 2>&1
tail -32 gpurun_out/r2i/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3

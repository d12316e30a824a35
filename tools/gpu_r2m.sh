mkdir -p gpurun_out/r2m
for n in 4 8; do
  timeout 900 python bench.py --simulate-bands $n --no-cpu-baseline --no-per-config --no-e2e > gpurun_out/r2m/bands$n.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2m/bands$n.json').read().strip().splitlines()[-1]); print('bands $n tuned', round(d['ms_per_step']*1e3,2), 'us', [(c['V'],c['TX'],c['TH']) for c in d['config']['schedule']])"
  for o in "vec=4,chunks=1,rows=16,warps=1,prefetch=4" "vec=2,chunks=1,rows=32,warps=1,prefetch=4" "vec=2,chunks=1,rows=16,warps=1,prefetch=4" "vec=4,chunks=1,rows=24,warps=1,prefetch=4" "vec=1,chunks=4,rows=16,warps=1,prefetch=4"; do
    timeout 600 python bench.py --simulate-bands $n --no-cpu-baseline --no-per-config --no-e2e --opts $o > gpurun_out/r2m/b.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r2m/b.json').read().strip().splitlines()[-1]); print('bands $n $o', round(d['ms_per_step']*1e3,2), 'us')"
  done
done
for o in "vec=4,chunks=1,rows=100,warps=1,prefetch=4" "vec=4,chunks=1,rows=100,warps=1,prefetch=3" "vec=4,chunks=1,rows=100,warps=2,prefetch=4" "vec=4,chunks=1,rows=96,warps=1,prefetch=4"; do
  bash tools/bench_variants.sh r2m harris ";$o"
done

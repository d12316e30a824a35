for m in 0 1 0 1; do
  PMG_XMERGE=$m timeout 300 python bench.py --no-cpu-baseline --no-per-config --no-e2e > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('XMERGE=$m harris', round(d['ms_per_step']*1e3,2), d['gpu_launches']//d['steps'])"
  PMG_XMERGE=$m timeout 300 python bench.py --workload unsharp --no-cpu-baseline --no-per-config --no-e2e > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('XMERGE=$m unsharp', round(d['ms_per_step']*1e3,2), d['gpu_launches']//d['steps'])"
done

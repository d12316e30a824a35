# bench.py lines for a list of schedule / environment variants: bash tools/bench_variants.sh <tag> <workload> <variant>...
# a variant is "ENV=v,ENV2=w;opts" (either part may be empty), e.g. "PMG_FENCE=1;vec=4,chunks=1,rows=96,warps=1,prefetch=4"
tag=$1; wl=$2; shift 2
mkdir -p gpurun_out/$tag
for v in "$@"; do
  envs=${v%%;*}; opts=${v#*;}
  [ "$envs" = "$v" ] && opts=""
  out=gpurun_out/$tag/$(echo "$wl-$v" | tr -c 'A-Za-z0-9_.=-' '_').json
  env $(echo $envs | tr ',' ' ') timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 50 --warmup 5 --no-e2e ${opts:+--opts $opts} > $out 2> $out.err
  python - "$out" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ks = d["config"].get("kernels", [{}])
    print(f"{sys.argv[2]:60s} {d['ms_per_step']*1e3:8.2f} us  hbm {d['roofline']['hbm']['frac']:.3f}  launches {d['gpu_launches']//d['steps']}  "
          f"regs {[k.get('regs') for k in ks]} edge {[k.get('edge_regs') for k in ks]} bdr {[k.get('border_regs') for k in ks]}  "
          + " | ".join(f"V{c['V']}TX{c['TX']}TH{c['TH']}NW{c['NW']}" for c in d['config']['schedule'][:6]))
except Exception as e:
    print(sys.argv[2], "FAILED", e, open(sys.argv[1] + ".err").read()[-600:])
PY
done

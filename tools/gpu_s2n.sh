# unsharp configuration grid (is there a schedule above 60 % of HBM at 2048^2 x 3?)
tag=s2n
mkdir -p gpurun_out/$tag
S=""
for v in 1 2 4; do for tx in 1 2 4; do for th in 16 24 32 48 64; do
  cw=$((32*v*tx)); if [ $cw -ge 32 ] && [ $cw -le 256 ]; then S="$S vec=$v,chunks=$tx,rows=$th,warps=1,prefetch=4"; fi
done; done; done
timeout 1200 python tools/sweep.py unsharp $S > gpurun_out/$tag/unsharp_grid.txt 2>&1
sort -t: -k3 -n gpurun_out/$tag/unsharp_grid.txt | head -3
python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/s2n/unsharp_grid.txt") if l.startswith("{") and '"ms"' in l]
rows.sort(key=lambda r: r["ms"])
for r in rows[:10]: print(r["spec"], r["ms"], r["GB/s"], r["kernels(regs,spill,blk/SM)"])
PY

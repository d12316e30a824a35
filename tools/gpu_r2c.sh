mkdir -p gpurun_out/r2c
O="vec=4,chunks=1,rows=96,warps=1,prefetch=4"
bash tools/bench_variants.sh r2c harris "PMG_FENCE=1;$O" ";$O" "PMG_DIAG_SKIP=be;$O" "PMG_DIAG_SKIP=ie;$O" "PMG_DIAG_SKIP=ib;$O" "PMG_DIAG_SKIP=be,PMG_FENCE=1;$O"
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/r2c/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-graph --opts $O > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r2c/launches.csv')) if len(r)>10]
hdr=rows[0]; i_n=hdr.index('Kernel Name'); i_m=hdr.index('Metric Name'); i_v=hdr.index('Metric Value'); i_id=hdr.index('ID')
from collections import defaultdict
d=defaultdict(dict)
for r in rows[1:]: d[(r[i_id], r[i_n])][r[i_m]]=r[i_v]
for k,v in list(d.items())[-12:]: print(k, v)
PY
for f in "" 1; do
PMG_FENCE=$f timeout 600 ncu --set full --clock-control none --import-source on -k regex:'pmg_g0$' -c 1 -o gpurun_out/r2c/harris_full_f$f python tools/run_once.py harris "$O" 2 > gpurun_out/r2c/ncu_full_f$f.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "operator" > gpurun_out/r2c/pytest.txt 2>&1; tail -2 gpurun_out/r2c/pytest.txt

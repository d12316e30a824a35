# x-border kernel for the N=8 band (x-border tiles through the interior bodies)
tag=s2u
mkdir -p gpurun_out/$tag
for xk in 0 4 8 16; do PMG_XK=$xk timeout 600 python bench.py --simulate-bands 8 --no-cpu-baseline > gpurun_out/$tag/bands8_xk$xk.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/$tag/bands8_xk$xk.json')); print($xk, d['ms_per_step'], d['gpu_launches'])"; done
for xk in 4 8; do PMG_XK=$xk timeout 600 python bench.py --simulate-bands 4 --no-cpu-baseline > gpurun_out/$tag/bands4_xk$xk.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/$tag/bands4_xk$xk.json')); print('N4', $xk, d['ms_per_step'])"; done

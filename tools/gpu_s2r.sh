# projected band scaling on one GPU (band N/2 of N timed alone), N = 2, 4, 8
tag=s2r
mkdir -p gpurun_out/$tag
for n in 2 4 8; do timeout 600 python bench.py --simulate-bands $n --no-cpu-baseline > gpurun_out/$tag/bands_$n.json 2> gpurun_out/$tag/bands_$n.err; done
for n in 2 4 8; do python -c "
import json; d=json.load(open('gpurun_out/$tag/bands_$n.json')); print($n, d['ms_per_step'], d['value'], d['config'].get('launch'))"; done

# N=8 band: border-tile height (the band's x-border kernel is its latency floor)
tag=s2s
mkdir -p gpurun_out/$tag
for bth in 4 8 16; do PMG_BORDER_TH=$bth timeout 600 python bench.py --simulate-bands 8 --no-cpu-baseline > gpurun_out/$tag/bands8_bth$bth.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/$tag/bands8_bth$bth.json')); print($bth, d['ms_per_step'])"; done
for bth in 4 8; do PMG_BORDER_TH=$bth timeout 600 python bench.py --no-cpu-baseline > gpurun_out/$tag/full_bth$bth.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/$tag/full_bth$bth.json')); print('full', $bth, d['ms_per_step'])"; done

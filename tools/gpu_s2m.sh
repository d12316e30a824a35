# final session check: full GPU suite, smoke, bench (auto launch mode / graph / host), ncu launch list + full capture
tag=s2m
mkdir -p gpurun_out/$tag
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/$tag/pytest_gpu.txt 2>&1; tail -3 gpurun_out/$tag/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$tag/smoke.txt 2>&1; tail -2 gpurun_out/$tag/smoke.txt
timeout 600 python bench.py --graph --no-cpu-baseline > gpurun_out/$tag/bench_graph.json 2> gpurun_out/$tag/bench_graph.err
timeout 600 python bench.py --no-graph --no-cpu-baseline > gpurun_out/$tag/bench_host.json 2> gpurun_out/$tag/bench_host.err
bash tools/gpu_profile.sh $tag
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/$tag/bench_reference.json 2> gpurun_out/$tag/bench_reference.err
for f in bench.json bench_graph.json bench_host.json bench_reference.json; do echo $f; python -c "
import json,sys; d=json.load(open('gpurun_out/$tag/$f')); print(d.get('ms_per_step'), d.get('value'), d.get('config',{}).get('launch'), d.get('roofline',{}).get('frac'))"; done

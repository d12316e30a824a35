# camera: ncu launch list + full capture of the tuned plan's kernels; Harris band projection at N = 2, 4, 8
mkdir -p gpurun_out/r2h
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h/launches_camera.csv \
  python tools/run_once.py camera tune=1 3 > gpurun_out/r2h/camera_run.log 2>&1
tail -2 gpurun_out/r2h/camera_run.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pmg_g -c 6 -o gpurun_out/r2h/camera_full \
  python tools/run_once.py camera "" 1 > gpurun_out/r2h/ncu_full.log 2>&1
tail -2 gpurun_out/r2h/ncu_full.log
for n in 2 4 8; do
  timeout 600 python bench.py --simulate-bands $n --no-cpu-baseline --no-per-config --no-e2e > gpurun_out/r2h/harris_b$n.json 2> gpurun_out/r2h/harris_b$n.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2h/harris_b$n.json').read().strip().splitlines()[-1]); print('bands $n', round(d['ms_per_step']*1e3,2), 'us', [(c['V'],c['TX'],c['TH'],c['PREF']) for c in d['config']['schedule']], d['config']['launch'])"
done

# one iteration: GPU tests, quick bench line, launch-list shares
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --steps 3 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print('value', round(d['value']/1e9,2), 'G/s  traj_ms', round(d['traj_kernel_ms'],1), 'ms/step', round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value']/1e9,2), 'frac', round(d['roofline']['frac'],3))
print('overlay', {k: d.get('overlay_latency_ms',{}).get(k) for k in ('cold','warm_steering')}, d.get('overlay_latency_ms',{}).get('node_ms_cold'))
PY
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-overlay"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu=$?

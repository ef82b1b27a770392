python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/final6_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/final6_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/final6_smoke.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final6_bench.json 2> gpurun_out/final6_bench.err; echo bench=$?
python -c "
import json; d = json.loads(open('gpurun_out/final6_bench.json').read().strip().splitlines()[-1])
print(round(d['value'] / 1e9, 2), round(d['traj_kernel_ms'], 2), d['clocks'], round(d['e2e']['value'] / 1e9, 2), d['overlay_latency_ms']['warm_steering'])"

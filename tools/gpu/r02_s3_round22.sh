# C5: long-first order on / off; then the pipelined bench at C3 (short)
BUILDS="-DWG_TRAJ_ORDER=1 -DWG_TRAJ_ORDER=0" REPS=3 PROBE_ARGS="--size 65536 --stride 128 --seed 2 --lattice" bash tools/gpu/ab_traj.sh
python bench.py --gpus 1 --steps 8 --warmup 3 --no-cpu --no-overlay > gpurun_out/pipe_bench.json 2> gpurun_out/pipe_bench.err; echo pipe=$?; tail -c 200 gpurun_out/pipe_bench.err
python bench.py --gpus 1 --steps 8 --warmup 3 --no-cpu --no-overlay --serial > gpurun_out/serial_bench.json 2> gpurun_out/serial_bench.err; echo serial=$?
python - <<'PY'
import json
for f in ("gpurun_out/pipe_bench.json", "gpurun_out/serial_bench.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, round(d["value"] / 1e9, 2), round(d["ms_per_step"], 2), round(d["traj_kernel_ms"], 2), d["clocks"]["sm_mhz"], round(d["e2e"]["value"] / 1e9, 2))
PY

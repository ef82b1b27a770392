# Code-path check of bench.py's N>1 path on ONE GPU: 2 ranks over gloo (NCCL
# refuses two ranks per device).  Small config; the numbers mean nothing.
WG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --size 4096 --stride 32 --ppc 256 \
  --steps 3 --warmup 2 --no-cpu --no-overlay > gpurun_out/mr.log 2> gpurun_out/mr.err
echo multirank=$?
tail -1 gpurun_out/mr.log | cut -c1-400
python bench.py --size 4096 --stride 32 --ppc 256 --steps 3 --warmup 2 --no-cpu --no-overlay > gpurun_out/sr.log 2>&1
echo single=$?
python - <<'PY'
import json
m = json.loads(open('gpurun_out/mr.log').read().strip().splitlines()[-1])
s = json.loads(open('gpurun_out/sr.log').read().strip().splitlines()[-1])
print("steps equal:", m["particle_steps_per_step"] == s["particle_steps_per_step"], m["particle_steps_per_step"])
PY

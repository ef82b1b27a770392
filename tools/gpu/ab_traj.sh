# A/B of trajectory-kernel variants on the bench workload (env switches), plus GPU tests
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-"WG_TRAJ_AGG=0" "WG_TRAJ_AGG=1"}; do
  env $v timeout 600 python bench.py --no-cpu --no-overlay --steps 3 > gpurun_out/ab.log 2>/dev/null
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print(round(d['value']/1e9,2),'Gsteps/s traj_ms',round(d['traj_kernel_ms'],1),'frac',round(d['roofline']['frac'],3))")"
done

# A/B of trajectory-kernel compile variants (NVCC_EXTRA) on the bench workload
for v in ${BUILDS:-"-DWG_TRAJ_MINBLOCKS=8" "-DWG_TRAJ_MINBLOCKS=7" "-DWG_TRAJ_MINBLOCKS=6"}; do
  make -C paper_2506_23364_b200/csrc clean >/dev/null
  make -C paper_2506_23364_b200/csrc -j8 NVCC_EXTRA="$v" >/dev/null 2>&1 || { echo "build $v failed"; continue; }
  timeout 600 python bench.py --no-cpu --no-overlay --steps 3 > gpurun_out/ab.log 2>gpurun_out/ab.err
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print(round(d['value']/1e9,2),'Gsteps/s traj_ms',round(d['traj_kernel_ms'],1))" 2>&1 | tail -1)" | tee -a gpurun_out/ab_results.txt
done
make -C paper_2506_23364_b200/csrc clean >/dev/null
make -C paper_2506_23364_b200/csrc -j8 >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log

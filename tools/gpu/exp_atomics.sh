# experiment: trajectory kernel time with atomics partially disabled (results invalid; timing only)
make -C paper_2506_23364_b200/csrc clean >/dev/null
make -C paper_2506_23364_b200/csrc -j8 NVCC_EXTRA=-DWG_EXPERIMENT_ATOMICS >/dev/null 2>&1 || exit 1
for v in "WG_ATOM_MODE=3" "WG_ATOM_MODE=1" "WG_ATOM_MODE=2" "WG_ATOM_MODE=0"; do
  env $v timeout 600 python bench.py --no-cpu --no-overlay --steps 3 > gpurun_out/ab.log 2>/dev/null
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('traj_ms',round(d['traj_kernel_ms'],1))" 2>&1 | tail -1)"
done
make -C paper_2506_23364_b200/csrc clean >/dev/null

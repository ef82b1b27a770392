# A/B of whole traj.cu variants (tools/gpu/variants/*.cu, VARIANTS env) on the
# bench workload, same box, interleaved twice to expose drift
cp paper_2506_23364_b200/csrc/traj.cu /tmp/traj_keep.cu
for round in 1 2 3; do
for v in ${VARIANTS:-$(ls tools/gpu/variants/*.cu)}; do
  cp "$v" paper_2506_23364_b200/csrc/traj.cu
  make -C paper_2506_23364_b200/csrc -j8 >/dev/null 2>&1 || { echo "build $v failed"; continue; }
  timeout 600 python bench.py --no-cpu --no-overlay --no-e2e --steps 6 > gpurun_out/ab.log 2>gpurun_out/ab.err
  echo "$round $v $(python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print(round(d['value']/1e9,2),'Gsteps/s traj_ms',round(d['traj_kernel_ms'],1),d['clocks'])" 2>&1 | tail -1)" | tee -a gpurun_out/ab_results.txt
done
done
cp /tmp/traj_keep.cu paper_2506_23364_b200/csrc/traj.cu
make -C paper_2506_23364_b200/csrc -j8 >/dev/null 2>&1

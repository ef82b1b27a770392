# A/B of trajectory-kernel compile variants (NVCC_EXTRA) with the in-process
# (a variant may hold several flags separated by commas)
# probe (REPS launches each; min and median ms), two interleaved rounds
for round in 1 2; do
for v in ${BUILDS:-"-DWG_TRAJ_MINBLOCKS=7"}; do
  make -C paper_2506_23364_b200/csrc clean >/dev/null
  make -C paper_2506_23364_b200/csrc -j8 NVCC_EXTRA="${v//,/ }" >/dev/null 2>&1 || { echo "build $v failed"; continue; }
  timeout 600 python tools/traj_probe.py --reps ${REPS:-6} > gpurun_out/ab.log 2>gpurun_out/ab.err
  echo "$round $v $(python -c "
import json,statistics as st
d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('min', min(d['ms']), 'med', st.median(d['ms']), 'G/s', d['gsteps_s_best'], 'mhz_min', min(c.get('mhz_min',0) for c in d['clocks']) if d['clocks'] else None)" 2>&1 | tail -1)" | tee -a gpurun_out/ab_results.txt
done
done
make -C paper_2506_23364_b200/csrc clean >/dev/null
make -C paper_2506_23364_b200/csrc -j8 >/dev/null 2>&1

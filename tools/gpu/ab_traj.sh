# A/B of trajectory-kernel compile variants: only traj.o is rebuilt per
# variant (NVCC_EXTRA; a variant's flags are comma-separated), then
# tools/traj_probe.py times REPS launches at C3 in one process; two
# interleaved rounds.  Results: gpurun_out/ab_traj.txt
C=paper_2506_23364_b200/csrc
for round in 1 2; do
for v in ${BUILDS}; do
  rm -f paper_2506_23364_b200/_lib/obj/traj.o
  make -C $C -j8 NVCC_EXTRA="${v//,/ }" >/dev/null 2>&1 || { echo "build $v failed"; continue; }
  timeout 600 python tools/traj_probe.py --reps ${REPS:-6} ${PROBE_ARGS:-} > gpurun_out/ab.log 2>gpurun_out/ab.err; grep -h "traj timing" gpurun_out/ab.err | tail -2 >> gpurun_out/ab_timing.txt
  echo "$round $v $(python -c "
import json,statistics as st
d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('min', min(d['ms']), 'med', st.median(d['ms']), 'G/s', d['gsteps_s_best'], 'chk', d['hits_wsum'], d['zbits_xor'], 'mhz', [c.get('mhz_med') for c in d['clocks']][:3])" 2>&1 | tail -1)" | tee -a gpurun_out/ab_traj.txt
done
done
rm -f paper_2506_23364_b200/_lib/obj/traj.o
make -C $C -j8 >/dev/null 2>&1

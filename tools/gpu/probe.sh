# per-launch trajectory timing distribution, per traj.cu variant
cp paper_2506_23364_b200/csrc/traj.cu /tmp/traj_keep.cu
first=1
for v in ${VARIANTS:-$(ls tools/gpu/variants/*.cu)}; do
  cp "$v" paper_2506_23364_b200/csrc/traj.cu
  make -C paper_2506_23364_b200/csrc -j8 >/dev/null 2>&1 || { echo "build $v failed"; continue; }
  extra=""; [ $first = 1 ] && extra="--records"; first=0
  echo "$v $(timeout 600 python tools/traj_probe.py --reps ${REPS:-8} $extra 2>&1 | tail -1)" | tee -a gpurun_out/probe.txt
done
cp /tmp/traj_keep.cu paper_2506_23364_b200/csrc/traj.cu
make -C paper_2506_23364_b200/csrc -j8 >/dev/null 2>&1

# drain tail at the C4 overlay config (diagnostic build), and the N>1 bench
# code path over gloo
rm -f paper_2506_23364_b200/_lib/obj/traj.o
make -C paper_2506_23364_b200/csrc -j8 NVCC_EXTRA="-DWG_TRAJ_TIMING=7" > /dev/null 2>&1
python tools/overlay_probe.py 8192 16 256 4 > gpurun_out/ov_timing.log 2>&1; grep -h "traj timing\|rep" gpurun_out/ov_timing.log | tail -6
timeout 600 python tools/traj_probe.py --reps 2 > /dev/null 2> gpurun_out/c3_timing.err; grep "traj timing" gpurun_out/c3_timing.err | tail -2
rm -f paper_2506_23364_b200/_lib/obj/traj.o
make -C paper_2506_23364_b200/csrc -j8 > /dev/null 2>&1
bash tools/gpu/multirank_gloo.sh

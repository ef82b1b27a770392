# where the trajectory launch's time goes: pool drain vs last warp (diagnostic
# build), single pass, then the two-pass at 7 blocks/SM (73 registers: no spill)
BUILDS="-DWG_TRAJ_TIMING=1 -DWG_TRAJ_TIMING=1,-DWG_TRAJ_BUDGET=512 -DWG_TRAJ_MINBLOCKS=7 -DWG_TRAJ_MINBLOCKS=7,-DWG_TRAJ_BUDGET=512" REPS=4 bash tools/gpu/ab_traj.sh
grep -h "traj timing" gpurun_out/ab.err | tail -3

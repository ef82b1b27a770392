# start-up dynamics of the persistent trajectory kernel: staggered warp
# starts, cell-interleaved claim order, the timestamp prologue; mip occupancy
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_TIMING=1 -DWG_TRAJ_STAGGER=50 -DWG_TRAJ_STAGGER=1000 -DWG_TRAJ_INTERLEAVE=1 -DWG_TRAJ_INTERLEAVE=1,-DWG_TRAJ_TIMING=1" REPS=5 bash tools/gpu/ab_traj.sh
BUILDS="-DWG_AB_DEFAULT=1 -DWG_MIP_MINB=5" REPS=20 bash tools/gpu/ab_tex.sh

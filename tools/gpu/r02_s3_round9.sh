# the diagnostic build ran faster than the default: which of its pieces
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_TIMING=7 -DWG_TRAJ_TIMING=1 -DWG_TRAJ_TIMING=2 -DWG_TRAJ_TIMING=4" REPS=6 bash tools/gpu/ab_traj.sh

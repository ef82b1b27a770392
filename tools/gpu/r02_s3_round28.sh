# release point in shared memory (not live across the loop) at 8 and 9 blocks/SM
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_RELSMEM=1 -DWG_TRAJ_RELSMEM=1,-DWG_TRAJ_MINBLOCKS=9" REPS=5 bash tools/gpu/ab_traj.sh

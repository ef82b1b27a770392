# is the diagnostic prologue's speed-up the step loop's placement? prologue
# padding 0..7 instructions (16 B each) vs the timestamp prologue
BUILDS="-DWG_TRAJ_PAD=0 -DWG_TRAJ_PAD=1 -DWG_TRAJ_PAD=2 -DWG_TRAJ_PAD=3 -DWG_TRAJ_PAD=4 -DWG_TRAJ_PAD=5 -DWG_TRAJ_PAD=6 -DWG_TRAJ_PAD=7 -DWG_TRAJ_TIMING=1" REPS=5 bash tools/gpu/ab_traj.sh

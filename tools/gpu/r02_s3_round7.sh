# two-pass trajectory launches (long particles suspended at a step budget in
# the first pass and resumed together in a second): A/B of budgets
BUILDS="-DWG_TRAJ_BUDGET=0 -DWG_TRAJ_BUDGET=256 -DWG_TRAJ_BUDGET=512 -DWG_TRAJ_BUDGET=1024" REPS=6 bash tools/gpu/ab_traj.sh

# C5 (L1/TEX-bound) with the red reductions: pair 256-bit loads off / on, the two-copy table
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_PAIRV4=0 -DWG_TRAJ_TAB2=1" REPS=3 PROBE_ARGS="--size 65536 --stride 128 --seed 2 --lattice" bash tools/gpu/ab_traj.sh

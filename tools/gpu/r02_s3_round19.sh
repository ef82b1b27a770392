BUILDS="-DWG_TRAJ_ORDER=0 -DWG_TRAJ_ORDER_T=32 -DWG_TRAJ_ORDER_T=32,-DWG_TRAJ_ORDER_P=4 -DWG_TRAJ_ORDER_T=16,-DWG_TRAJ_ORDER_P=4" REPS=10 PROBE_ARGS="--size 8192 --seed 1 --stride 16 --ppc 256" bash tools/gpu/ab_traj.sh
mv gpurun_out/ab_traj.txt gpurun_out/ab_traj_c4.txt
BUILDS="-DWG_TRAJ_ORDER=0 -DWG_TRAJ_ORDER_T=32 -DWG_TRAJ_ORDER_T=32,-DWG_TRAJ_ORDER_P=4" REPS=4 bash tools/gpu/ab_traj.sh

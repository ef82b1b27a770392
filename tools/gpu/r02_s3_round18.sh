# longest-first order as a stable two-bucket partition (thresholds 32 / 64 / 128 probe steps)
python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/s3r18_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/s3r18_tests.log
BUILDS="-DWG_TRAJ_ORDER=0 -DWG_TRAJ_ORDER_T=128 -DWG_TRAJ_ORDER_T=64 -DWG_TRAJ_ORDER_T=32" REPS=10 PROBE_ARGS="--size 8192 --seed 1 --stride 16 --ppc 256" bash tools/gpu/ab_traj.sh
mv gpurun_out/ab_traj.txt gpurun_out/ab_traj_c4.txt
BUILDS="-DWG_TRAJ_ORDER=0 -DWG_TRAJ_ORDER_T=128 -DWG_TRAJ_ORDER_T=32" REPS=4 bash tools/gpu/ab_traj.sh

# gather layout as a template parameter (each kernel carries only its own
# gather) and, for the row-pair layout (C5), one 256-bit load for even patches
python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py -q -x -p no:cacheprovider > gpurun_out/s3r20_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/s3r20_tests.log
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_LAYOUT_T=0" REPS=5 bash tools/gpu/ab_traj.sh
mv gpurun_out/ab_traj.txt gpurun_out/ab_traj_c3.txt
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_PAIRV4=0 -DWG_TRAJ_LAYOUT_T=0" REPS=3 PROBE_ARGS="--size 65536 --stride 128 --seed 2 --lattice" bash tools/gpu/ab_traj.sh

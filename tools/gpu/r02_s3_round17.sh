# longest-first release-cell order: parity, then A/B at C4 (overlay config) and C3
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_stress.py -q -x -p no:cacheprovider > gpurun_out/s3r17_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/s3r17_tests.log
BUILDS="-DWG_TRAJ_ORDER=1 -DWG_TRAJ_ORDER=0" REPS=10 PROBE_ARGS="--size 8192 --seed 1 --stride 16 --ppc 256" bash tools/gpu/ab_traj.sh
mv gpurun_out/ab_traj.txt gpurun_out/ab_traj_c4.txt
BUILDS="-DWG_TRAJ_ORDER=1 -DWG_TRAJ_ORDER=0" REPS=5 bash tools/gpu/ab_traj.sh
python tools/overlay_probe.py 8192 16 256 4 > gpurun_out/s3r17_ov.log 2>&1; tail -2 gpurun_out/s3r17_ov.log

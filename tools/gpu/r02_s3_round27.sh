# with the PTX red reductions: is the CTA-start counter still worth it; the drop max unconditional
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_CTA_COUNT=0 -DWG_TRAJ_ZMAX_UNCOND=1" REPS=5 bash tools/gpu/ab_traj.sh
mv gpurun_out/ab_traj.txt gpurun_out/ab_traj_c3.txt
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_CTA_COUNT=0" REPS=10 PROBE_ARGS="--size 8192 --seed 1 --stride 16 --ppc 256" bash tools/gpu/ab_traj.sh
python -m pytest tests/test_gpu_multirank.py tests/test_gpu_c5.py -q -x -p no:cacheprovider > gpurun_out/s3r27_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/s3r27_tests.log

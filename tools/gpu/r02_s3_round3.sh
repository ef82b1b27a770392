# trajectory kernel: branch hints, one stop branch, trig constants in the
# parameter block -- parity at the default build, then the A/B
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/s3r3_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/s3r3_tests.log
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_EXPECT=0 -DWG_TRAJ_ONESTOP=0 -DWG_TRAJ_TC_PARAM=0 -DWG_TRAJ_EXPECT=0,-DWG_TRAJ_ONESTOP=0,-DWG_TRAJ_TC_PARAM=0" REPS=6 bash tools/gpu/ab_traj.sh

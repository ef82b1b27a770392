# the raster reductions as PTX red (REDG; the drop under a predicate) vs atomicAdd / atomicMax (ATOMG to RZ)
rm -f paper_2506_23364_b200/_lib/obj/traj.o; make -C paper_2506_23364_b200/csrc -j8 NVCC_EXTRA="-DWG_TRAJ_PRED_RED=1" > /dev/null 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -q -x -p no:cacheprovider > gpurun_out/s3r26_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/s3r26_tests.log
BUILDS="-DWG_TRAJ_PRED_RED=0 -DWG_TRAJ_PRED_RED=1" REPS=5 bash tools/gpu/ab_traj.sh
mv gpurun_out/ab_traj.txt gpurun_out/ab_traj_c3.txt
BUILDS="-DWG_TRAJ_PRED_RED=0 -DWG_TRAJ_PRED_RED=1" REPS=10 PROBE_ARGS="--size 8192 --seed 1 --stride 16 --ppc 256" bash tools/gpu/ab_traj.sh

# two-particles-per-thread trajectory kernel: parity under that build, then A/B
make -C paper_2506_23364_b200/csrc clean >/dev/null
make -C paper_2506_23364_b200/csrc -j8 NVCC_EXTRA="-DWG_TRAJ_PAIR=1" >/dev/null 2>&1 || echo BUILD FAILED
python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_fullsize.py tests/test_gpu_baseline_configs.py tests/test_gpu_c5.py -q -x -p no:cacheprovider > gpurun_out/t10.log 2>&1; tail -5 gpurun_out/t10.log
BUILDS="-DWG_TRAJ_PAIR=0 -DWG_TRAJ_PAIR=1 -DWG_TRAJ_PAIR=1,-DWG_TRAJ_PAIR_MINBLOCKS=3 -DWG_TRAJ_PAIR=1,-DWG_TRAJ_PAIR_MINBLOCKS=5" REPS=5 bash tools/gpu/ab_build.sh

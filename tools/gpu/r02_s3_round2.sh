# parity of the changed kernels (trajectory: jitter draw from bits, one vote
# per step, no large-argument sincos branch; textures: integer mip path,
# select-free colorize), then the trajectory A/B and texture ncu captures
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_c4_full.py tests/test_gpu_hillshade.py tests/test_gpu_tiles.py tests/test_gpu_baseline_configs.py tests/test_gpu_stress.py tests/test_gpu_trig_gate.py -q -x -p no:cacheprovider > gpurun_out/s3r2_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/s3r2_tests.log
python tools/overlay_probe.py > gpurun_out/s3r2_ov.log 2>&1; echo probe=$?; tail -2 gpurun_out/s3r2_ov.log
for K in colorize_kernel mip_tile_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_s3r2_$K -f python tools/overlay_probe.py > gpurun_out/ncu_$K.log 2>&1; echo ncu $K=$?
done
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_ONEVOTE=0,-DWG_TRAJ_U2BITS=0,-DWG_TRAJ_SMALLJIT=0 -DWG_TRAJ_ONEVOTE=0 -DWG_TRAJ_U2BITS=0 -DWG_TRAJ_SMALLJIT=0 -DWG_TRAJ_SAMPLE_REDO=1" REPS=6 bash tools/gpu/ab_traj.sh

# texture kernels after the select-free colorize and the integer mip path:
# parity tests that cover them, then one ncu --set full capture each
python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py tests/test_gpu_c4_full.py tests/test_gpu_tiles.py tests/test_gpu_hillshade.py -q -x -p no:cacheprovider > gpurun_out/s3_tex_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/s3_tex_tests.log
python tools/overlay_probe.py > gpurun_out/s3_plain_ov.log 2>&1; echo probe=$?; tail -3 gpurun_out/s3_plain_ov.log
for K in colorize_kernel mip_tile_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_s3_$K -f python tools/overlay_probe.py > gpurun_out/ncu_$K.log 2>&1; echo ncu $K=$?
done

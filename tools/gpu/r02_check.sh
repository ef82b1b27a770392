python -m pytest tests/test_gpu_slope.py tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py tests/test_gpu_hillshade.py -q -x -p no:cacheprovider > gpurun_out/t11.log 2>&1; tail -3 gpurun_out/t11.log
python tools/bench_stencil.py > gpurun_out/stencil3.json 2>&1; cat gpurun_out/stencil3.json
python tools/overlay_probe.py > gpurun_out/plain_ov4.log 2>&1; tail -1 gpurun_out/plain_ov4.log
for K in colorize_kernel mip_tile_kernel; do
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_r02d_$K -f python tools/overlay_probe.py > /dev/null 2>&1; echo ncu $K=$?
done
ncu --set full --clock-control none --import-source on -k regex:normals_kernel -c 1 -o gpurun_out/prof_r02_normals -f python tools/bench_stencil.py > /dev/null 2>&1; echo ncu normals=$?

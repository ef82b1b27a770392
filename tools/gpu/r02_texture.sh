# round-2 texture kernels: parity tests, bench (e2e check), then one ncu
# --set full capture each of colorize_kernel and mip_tile_kernel
python -m pytest tests/test_gpu_ascii.py tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -q -x -p no:cacheprovider > gpurun_out/t6.log 2>&1; tail -3 gpurun_out/t6.log
python bench.py --steps 3 --warmup 3 --no-cpu --no-overlay > gpurun_out/b6.json 2> gpurun_out/b6.err; tail -c 600 gpurun_out/b6.json
python tools/overlay_probe.py > gpurun_out/plain_ov.log 2>&1 || tail gpurun_out/plain_ov.log
for K in colorize_kernel mip_tile_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_r02_$K -f python tools/overlay_probe.py > gpurun_out/ncu_$K.log 2>&1; echo ncu $K=$?
done

python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -q -x -p no:cacheprovider -k "colorize or c4 or executor" > gpurun_out/t13.log 2>&1; tail -2 gpurun_out/t13.log
python tools/overlay_probe.py > gpurun_out/plain_ov5.log 2>&1; tail -1 gpurun_out/plain_ov5.log
ncu --set full --clock-control none --import-source on -k regex:colorize_kernel -s 1 -c 1 -o gpurun_out/prof_r02f_colorize_kernel -f python tools/overlay_probe.py > /dev/null 2>&1; echo ncu colorize=$?

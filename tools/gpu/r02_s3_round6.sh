python -m pytest tests/test_gpu_parity.py tests/test_gpu_c4_full.py -q -x -p no:cacheprovider -k "colorize or c4 or mipmap" > gpurun_out/s3r6_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/s3r6_tests.log
python tools/overlay_probe.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:colorize_kernel -s 1 -c 1 -o gpurun_out/prof_s3r6_colorize -f python tools/overlay_probe.py > gpurun_out/ncu_colorize_kernel.log 2>&1; echo ncu=$?
timeout 900 python tools/traj_probe.py --reps 2 --records > gpurun_out/lifetimes.json 2> gpurun_out/lifetimes.err; echo rec=$?; cat gpurun_out/lifetimes.json; tail -3 gpurun_out/lifetimes.err

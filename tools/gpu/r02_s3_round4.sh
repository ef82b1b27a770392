# colorize with hoisted divisor / sign tests and one vote per four texels;
# trajectory pair-aggregated atomics (A/B)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_c4_full.py tests/test_gpu_baseline_configs.py -q -x -p no:cacheprovider -k "colorize or c4 or overlay or C4 or mipmap" > gpurun_out/s3r4_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/s3r4_tests.log
python tools/overlay_probe.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:colorize_kernel -s 1 -c 1 -o gpurun_out/prof_s3r4_colorize -f python tools/overlay_probe.py > gpurun_out/ncu_colorize_kernel.log 2>&1; echo ncu=$?
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_PAIRAGG=1" REPS=6 bash tools/gpu/ab_traj.sh
python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/s3r4_tests2.log 2>&1; echo tests2=$?; tail -2 gpurun_out/s3r4_tests2.log

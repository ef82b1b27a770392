# round-2 measurement set: tests of the touched kernels, the headline bench
# (driver parameters), the reference arm, C5, the launch list and one ncu
# --set full capture of the trajectory kernel
python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -q -x -p no:cacheprovider > gpurun_out/t12.log 2>&1; tail -2 gpurun_out/t12.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; tail -c 300 gpurun_out/r02_bench.json; tail -3 gpurun_out/r02_bench.err
python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2>&1; tail -c 300 gpurun_out/r02_bench_reference.json
python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/r02_bench_c5.json 2>&1; tail -c 300 gpurun_out/r02_bench_c5.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-overlay --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 1 -c 1 -o gpurun_out/prof_r02_traj -f python bench.py --steps 1 --warmup 1 --no-cpu --no-overlay --no-e2e > gpurun_out/ncu_traj.log 2>&1; echo ncu traj=$?
python tools/overlay_probe.py > /dev/null 2>&1; ncu --set full --clock-control none --import-source on -k regex:colorize_kernel -s 1 -c 1 -o gpurun_out/prof_r02e_colorize_kernel -f python tools/overlay_probe.py > /dev/null 2>&1; echo ncu colorize=$?

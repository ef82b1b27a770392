python bench.py --config c5 --steps 1 --warmup 1 --no-cpu --no-overlay --no-e2e > gpurun_out/c5_plain.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 1 -c 1 -o gpurun_out/prof_c5_traj -f python bench.py --config c5 --steps 1 --warmup 1 --no-cpu --no-overlay --no-e2e > gpurun_out/ncu_c5.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_c5.log

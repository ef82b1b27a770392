# profiles at the exact final build: launch list, ncu of the trajectory launch, C5 bench
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02j_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-overlay --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 1 -c 1 -o gpurun_out/prof_r02j_traj -f python bench.py --steps 1 --warmup 1 --no-cpu --no-overlay --no-e2e > gpurun_out/ncu_traj.log 2>&1; echo ncu=$?
python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/r02j_bench_c5.json 2>&1; echo c5=$?; tail -c 200 gpurun_out/r02j_bench_c5.json

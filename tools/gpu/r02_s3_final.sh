# round-2 final measurement set at the current build
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; echo bench=$?; tail -c 400 gpurun_out/r02i_bench.json; tail -3 gpurun_out/r02i_bench.err
python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/r02i_bench_reference.json 2>&1; echo ref=$?; tail -c 300 gpurun_out/r02i_bench_reference.json
python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/r02i_bench_c5.json 2>&1; echo c5=$?; tail -c 300 gpurun_out/r02i_bench_c5.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02i_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-overlay --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 1 -c 1 -o gpurun_out/prof_r02i_traj -f python bench.py --steps 1 --warmup 1 --no-cpu --no-overlay --no-e2e > gpurun_out/ncu_traj.log 2>&1; echo ncu traj=$?
python tools/overlay_probe.py > /dev/null 2>&1
for K in colorize_kernel mip_tile_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_r02i_$K -f python tools/overlay_probe.py > gpurun_out/ncu_$K.log 2>&1; echo ncu $K=$?
done
python tools/tex_probe.py > gpurun_out/r02i_tex.json 2>&1; tail -1 gpurun_out/r02i_tex.json

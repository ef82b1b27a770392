python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=8 > gpurun_out/t9.log 2>&1; tail -14 gpurun_out/t9.log
python tools/shard_probe.py --config c3 --world 2 --reps 2 > gpurun_out/sprobe2_c3.json 2>&1; cat gpurun_out/sprobe2_c3.json
python tools/shard_sim.py --config c3 > gpurun_out/shard2_c3.json 2> gpurun_out/shard2_c3.err; cat gpurun_out/shard2_c3.err
python tools/shard_sim.py --config c5 > gpurun_out/shard2_c5.json 2> gpurun_out/shard2_c5.err; cat gpurun_out/shard2_c5.err
python tools/overlay_probe.py > gpurun_out/plain_ov3.log 2>&1; cat gpurun_out/plain_ov3.log
ncu --set full --clock-control none --import-source on -k regex:colorize_kernel -s 1 -c 1 -o gpurun_out/prof_r02c_colorize_kernel -f python tools/overlay_probe.py > /dev/null 2>&1; echo ncu=$?
BUILDS="-DWG_TRAJ_TABREG=0 -DWG_TRAJ_TABREG=1 -DWG_TRAJ_TABREG=1,-DWG_TRAJ_ZMAX_UNCOND=1" REPS=5 bash tools/gpu/ab_build.sh

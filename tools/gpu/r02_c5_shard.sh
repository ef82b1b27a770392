python -m pytest tests/test_gpu_c5.py -q -x -p no:cacheprovider --durations=5 > gpurun_out/t7.log 2>&1; tail -8 gpurun_out/t7.log
python tools/shard_sim.py --config c3 > gpurun_out/shard_c3.json 2> gpurun_out/shard_c3.err; tail -c 400 gpurun_out/shard_c3.json; tail -3 gpurun_out/shard_c3.err
python tools/shard_sim.py --config c5 > gpurun_out/shard_c5.json 2> gpurun_out/shard_c5.err; tail -c 400 gpurun_out/shard_c5.json; tail -3 gpurun_out/shard_c5.err
python tools/bench_stencil.py > gpurun_out/stencil2.json 2>&1; cat gpurun_out/stencil2.json
python tools/overlay_probe.py > gpurun_out/plain_ov2.log 2>&1; cat gpurun_out/plain_ov2.log
ncu --set full --clock-control none --import-source on -k regex:colorize_kernel -s 1 -c 1 -o gpurun_out/prof_r02b_colorize_kernel -f python tools/overlay_probe.py > /dev/null 2>&1; echo ncu=$?

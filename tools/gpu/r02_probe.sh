python tools/shard_probe.py --config c3 --world 2 > gpurun_out/sprobe_c3.json 2>&1; cat gpurun_out/sprobe_c3.json
python tools/shard_probe.py --config c5 --world 2 --reps 2 > gpurun_out/sprobe_c5.json 2>&1; cat gpurun_out/sprobe_c5.json

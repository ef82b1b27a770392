set -x
timeout 900 python bench.py > gpurun_out/bench_full.log 2>gpurun_out/bench_full.err; echo bench=$?
tail -2 gpurun_out/bench_full.log
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-overlay"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu.log

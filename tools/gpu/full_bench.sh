# Round-end style measurement: reference arm, our arm (default flags), launch list
set -x
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo ref=$?
tail -1 gpurun_out/bench_ref.log | cut -c1-600
timeout 900 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo bench=$?
tail -1 gpurun_out/bench_full.log
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-overlay"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu=$?

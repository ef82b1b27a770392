# session-3 re-entry check: the whole GPU suite at HEAD, then the headline bench
python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/s3_gpu_tests.log 2>&1; echo tests=$?; tail -25 gpurun_out/s3_gpu_tests.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo bench=$?; tail -c 400 gpurun_out/s3_bench.json; tail -3 gpurun_out/s3_bench.err

# config 5 (65536^2, stride 128, 2048 ppc) on one GPU, plus GPU tests
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2> gpurun_out/bench_c5.err; echo c5=$?
tail -1 gpurun_out/bench_c5.log | cut -c1-900; tail -3 gpurun_out/bench_c5.err

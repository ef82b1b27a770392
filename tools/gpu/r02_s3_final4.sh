# the whole GPU suite (incl. the claim-order test) + smoke at the final build
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/final4_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/final4_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final4_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/final4_smoke.log
python bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --no-overlay > gpurun_out/final4_bench.json 2>&1; echo bench=$?; tail -c 300 gpurun_out/final4_bench.json

# round-2 final: the whole GPU suite + smoke at the final build, then the measurement set
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/final_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/final_smoke.log
bash tools/gpu/r02_s3_final.sh

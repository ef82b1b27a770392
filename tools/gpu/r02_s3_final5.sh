# final build (PTX red reductions): the whole GPU suite + smoke, the L2 probe, the measurement set
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/final5_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/final5_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final5_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/final5_smoke.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/l2_peak tools/micro/l2_peak.cu && ./tools/micro/l2_peak > gpurun_out/l2_peak2.json 2>&1; echo l2=$?; cat gpurun_out/l2_peak2.json
bash tools/gpu/r02_s3_final.sh

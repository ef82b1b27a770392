# Round-end measurement set: GPU tests + smoke, reference arm, full bench,
# launch list, ncu --set full of the trajectory kernel.
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 900 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo bench=$?
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-overlay"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo launches=$?
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-overlay --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 1 -c 1 -o gpurun_out/prof_traj -f $CMD > gpurun_out/ncu_prof.log 2>&1; echo ncu_full=$?

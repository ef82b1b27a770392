# ncu --set full capture of the trajectory kernel on the bench workload
set -x
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-overlay ${BENCH_ARGS:-}"
$CMD > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s ${SKIP:-1} -c 1 \
    -o gpurun_out/prof_traj -f $CMD > gpurun_out/ncu_prof.log 2>&1
echo ncu=$?
tail -3 gpurun_out/ncu_prof.log

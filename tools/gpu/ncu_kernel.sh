# ncu --set full of one kernel (regex K) on the bench workload
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-overlay ${BENCH_ARGS:-}"
$CMD > gpurun_out/plain_k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${K} -s ${SKIP:-1} -c 1 \
    -o gpurun_out/prof_${K} -f $CMD > gpurun_out/ncu_k.log 2>&1
echo ncu=$?

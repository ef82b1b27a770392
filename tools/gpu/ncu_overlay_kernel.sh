CMD="python tools/overlay_probe.py"
$CMD > gpurun_out/plain_ov.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:${K} -s ${SKIP:-1} -c 1 -o gpurun_out/prof_${K} -f $CMD > gpurun_out/ncu_ovk.log 2>&1; echo ncu=$?

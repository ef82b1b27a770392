CMD="python tools/overlay_probe.py"
$CMD > gpurun_out/overlay_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/overlay_launches.csv $CMD > gpurun_out/ncu_ov.log 2>&1; echo ncu=$?
cat gpurun_out/overlay_plain.log

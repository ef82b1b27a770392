# measurement set at the current build: L2 probe, ncu of the trajectory
# kernel (C3) and the texture kernels, the headline bench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/l2_peak tools/micro/l2_peak.cu && ./tools/micro/l2_peak > gpurun_out/l2_peak.json 2>&1; echo l2=$?; cat gpurun_out/l2_peak.json
python bench.py --steps 1 --warmup 1 --no-cpu --no-overlay > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 1 -c 1 -o gpurun_out/prof_s3_traj -f python bench.py --steps 1 --warmup 1 --no-cpu --no-overlay > gpurun_out/ncu_prof.log 2>&1; echo ncu traj=$?
python tools/overlay_probe.py > /dev/null 2>&1
for K in colorize_kernel mip_tile_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_s3m_$K -f python tools/overlay_probe.py > gpurun_out/ncu_$K.log 2>&1; echo ncu $K=$?
done
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s3m_bench.json 2> gpurun_out/s3m_bench.err; echo bench=$?; tail -c 300 gpurun_out/s3m_bench.json

# GPU tests, then the in-process trajectory probe and the A/B builds (BUILDS)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python tools/traj_probe.py --reps 6 | tee gpurun_out/probe.txt
[ -n "$BUILDS" ] && bash tools/gpu/ab_build.sh

# the CTA-start counter prologue vs none; then the whole GPU suite and smoke()
BUILDS="-DWG_AB_DEFAULT=1 -DWG_TRAJ_CTA_COUNT=0" REPS=5 bash tools/gpu/ab_traj.sh
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s3r13_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/s3r13_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3r13_smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/s3r13_smoke.log

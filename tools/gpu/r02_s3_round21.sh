# long-first order for banded (multi-range) launches: parity of the sharded
# paths, then the one-GPU shard simulation at C3 with and without the order
python -m pytest tests/test_gpu_multirank.py tests/test_gpu_c5.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/s3r21_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/s3r21_tests.log
python tools/shard_sim.py --config c3 --ns 2,4,8 > gpurun_out/shard_order1.json 2> gpurun_out/shard_order1.err; echo sim1=$?
rm -f paper_2506_23364_b200/_lib/obj/traj.o; make -C paper_2506_23364_b200/csrc -j8 NVCC_EXTRA="-DWG_TRAJ_ORDER=0" > /dev/null 2>&1
python tools/shard_sim.py --config c3 --ns 2,4,8 > gpurun_out/shard_order0.json 2> gpurun_out/shard_order0.err; echo sim0=$?
rm -f paper_2506_23364_b200/_lib/obj/traj.o; make -C paper_2506_23364_b200/csrc -j8 > /dev/null 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/shard_order1.json", "gpurun_out/shard_order0.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, "1gpu", round(d["one_gpu_traj_ms"], 1), {n: (s["max_rank_traj_ms"], s["traj_efficiency"]) for n, s in d["splits"].items()})
PY

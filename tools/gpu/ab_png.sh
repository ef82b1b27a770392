# A/B of PNG encoder compile variants (BUILDS = NVCC_EXTRA values) on the tile bench
# (a variant may hold several flags separated by commas)
for v in ${BUILDS:-"-DWG_PNG_RING=16" "-DWG_PNG_RING=26"}; do
  make -C paper_2506_23364_b200/csrc clean >/dev/null
  make -C paper_2506_23364_b200/csrc -j8 NVCC_EXTRA="${v//,/ }" >/dev/null 2>&1 || { echo "build $v failed"; continue; }
  timeout 600 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pt.log 2>&1 || { echo "$v tests FAILED"; tail -5 gpurun_out/pt.log; }
  timeout 600 python tools/bench_tiles.py --sample 20 > gpurun_out/tb.json 2>/dev/null
  echo "$v $(python -c "
import json; d=json.load(open('gpurun_out/tb.json'))
print({k: (round(d[k]['kernel_ms'],1), round(d[k]['mean_png_bytes']/1e3,1)) for k in ('hillshade','overlay')})")" | tee -a gpurun_out/ab_png.txt
done
make -C paper_2506_23364_b200/csrc clean >/dev/null
make -C paper_2506_23364_b200/csrc -j8 >/dev/null 2>&1

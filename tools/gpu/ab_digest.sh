# A/B of digest-kernel compile variants (NVCC_EXTRA, comma-separated flags)
for v in ${BUILDS:-"-DWG_DIGEST_UNROLL=8"}; do
  make -C paper_2506_23364_b200/csrc clean >/dev/null
  make -C paper_2506_23364_b200/csrc -j8 NVCC_EXTRA="${v//,/ }" >/dev/null 2>&1 || { echo "build $v failed"; continue; }
  echo "$v $(python tools/bench_digest.py 2>&1 | tail -1)"
done
make -C paper_2506_23364_b200/csrc clean >/dev/null
make -C paper_2506_23364_b200/csrc -j8 >/dev/null 2>&1

# A/B of texture-kernel compile variants: only texture.o is rebuilt per
# variant, then tools/tex_probe.py; two interleaved rounds -> gpurun_out/ab_tex.txt
C=paper_2506_23364_b200/csrc
for round in 1 2; do
for v in ${BUILDS}; do
  rm -f paper_2506_23364_b200/_lib/obj/texture.o
  make -C $C -j8 NVCC_EXTRA="${v//,/ }" >/dev/null 2>&1 || { echo "build $v failed"; continue; }
  echo "$round $v $(timeout 600 python tools/tex_probe.py --reps ${REPS:-20} 2>gpurun_out/ab_tex.err | tail -1)" | tee -a gpurun_out/ab_tex.txt
done
done
rm -f paper_2506_23364_b200/_lib/obj/texture.o
make -C $C -j8 >/dev/null 2>&1

# A/B: which part of the leaner fp64 epilogue helps / hurts: ldsonly (shared-space pointers only),
# clamponly (integer clamp + diagonal only), epi2 (both), cur (neither); bench loop (product, predict), C2.
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
for i in 1 2; do for v in ab/cur.so ab/ldsonly.so ab/clamponly.so ab/epi2.so; do
  PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/ab_step.py C1 12
done; done > gpurun_out/ab13.log 2>&1
for i in 1 2; do for v in ab/cur.so ab/ldsonly.so ab/clamponly.so ab/epi2.so; do
  echo -n "$v C2: "; PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/run_matvec.py --config C2 --synth --repeats 8
done; done >> gpurun_out/ab13.log 2>&1

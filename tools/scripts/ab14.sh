# A/B: 16-entry exp table + degree-7 polynomial (conflict-free table lookups, +3 DFMA / entry) vs the
# 256-entry table + degree 4 (current); C1 products, bench loop; the fp64 tests on the variant.
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
for i in 1 2 3; do for v in ab/cur2.so ab/exp16.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1000
done; done > gpurun_out/ab14.log 2>&1
for i in 1 2; do for v in ab/cur2.so ab/exp16.so; do
  PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/ab_step.py C1 12
done; done >> gpurun_out/ab14.log 2>&1
PLSSVM_LIB_PATH=$L/ab/exp16.so timeout 900 python -m pytest tests/test_gpu_fp64_engines.py -x -q > gpurun_out/ab14_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab14_tests.log

# A/B: leaner fp64 epilogue (shared-space pointers -> LDS, clamp + diagonal by integer masks, underflow
# test on the high word) vs the current build; C1 standalone products (sustained), C1 bench loop, C2;
# then the fp64 / parity tests.
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
for i in 1 2 3; do for v in ab/cur.so ab/epi2.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1000
done; done > gpurun_out/ab12.log 2>&1
for i in 1 2; do for v in ab/cur.so ab/epi2.so; do
  PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/ab_step.py C1 15
done; done >> gpurun_out/ab12.log 2>&1
for v in ab/cur.so ab/epi2.so; do
  echo -n "$v C2: "; PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/run_matvec.py --config C2 --synth --repeats 10
done >> gpurun_out/ab12.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fp64_engines.py tests/test_gpu_parity.py -x -q > gpurun_out/ab12_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab12_tests.log

# A/B: fp64 pass order big-first (levels 3-6 with all 7 planes, then levels 0-2 with 3 planes: 10 plane
# loads per slab instead of 11) vs the current order; correctness on the variant first.
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
PLSSVM_LIB_PATH=$L/ab/order10.so timeout 900 python -m pytest tests/test_gpu_fp64_engines.py -x -q > gpurun_out/ab16_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab16_tests.log
for i in 1 2 3; do for v in ab/cur3.so ab/order10.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1000
done; done > gpurun_out/ab16.log 2>&1
for i in 1 2; do for v in ab/cur3.so ab/order10.so; do
  PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/ab_step.py C1 12
done; done >> gpurun_out/ab16.log 2>&1
for i in 1 2; do for v in ab/cur3.so ab/order10.so; do
  echo -n "$v C2: "; PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/run_matvec.py --config C2 --synth --repeats 8
done; done >> gpurun_out/ab16.log 2>&1

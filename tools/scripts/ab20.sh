# A/B: fp32 engine 4 slabs per stage (two 2-slab boxes per operand; 3 or 2 stages of 72 KiB) vs 2 slabs (4 stages)
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
PLSSVM_LIB_PATH=$L/ab/s4st3.so timeout 900 python -m pytest tests/test_gpu_fp32_ozaki.py -x -q > gpurun_out/ab20_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab20_tests.log
PLSSVM_LIB_PATH=$L/ab/cur6.so timeout 900 python -m pytest tests/test_gpu_fp32_ozaki.py -x -q >> gpurun_out/ab20_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab20_tests.log
for i in 1 2 3; do for v in ab/cur6.so ab/s4st3.so ab/s4st2.so; do
  echo -n "$v C3: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 400
done; done > gpurun_out/ab20.log 2>&1

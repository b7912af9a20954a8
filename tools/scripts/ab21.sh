# A/B: bigger pipeline stages for the fp64 engine (2 slabs per stage in both passes / pass 1 only, 2 stages
# of 84 KiB) vs 1 slab (5 stages of 42 KiB); fp32 tests on the 4-slab / 2-stage variant
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
PLSSVM_LIB_PATH=$L/ab/s4st2.so timeout 900 python -m pytest tests/test_gpu_fp32_ozaki.py -x -q > gpurun_out/ab21_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab21_tests.log
PLSSVM_LIB_PATH=$L/ab/f64s2.so timeout 900 python -m pytest tests/test_gpu_fp64_engines.py -x -q >> gpurun_out/ab21_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab21_tests.log
for i in 1 2 3; do for v in ab/cur6.so ab/f64s2.so ab/f64s2p1.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1000
done; done > gpurun_out/ab21.log 2>&1

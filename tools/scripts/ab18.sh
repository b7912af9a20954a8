# A/B: fp64 engine pass 0 (4 planes) with 2 slabs per stage (4 stages of 48 KiB) vs 1 slab (5 of 42 KiB);
# correctness of both builds (fp64 / fp32 engine tests), C1 / C2 products, C3 on the current build.
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
PLSSVM_LIB_PATH=$L/ab/p0s2.so timeout 900 python -m pytest tests/test_gpu_fp64_engines.py -x -q > gpurun_out/ab18_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab18_tests.log
PLSSVM_LIB_PATH=$L/ab/cur5.so timeout 900 python -m pytest tests/test_gpu_fp32_ozaki.py tests/test_gpu_fp64_engines.py -x -q >> gpurun_out/ab18_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab18_tests.log
for i in 1 2 3; do for v in ab/cur5.so ab/p0s2.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1000
done; done > gpurun_out/ab18.log 2>&1
for v in ab/cur5.so ab/p0s2.so; do
  echo -n "$v C2: "; PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/run_matvec.py --config C2 --synth --repeats 8
done >> gpurun_out/ab18.log 2>&1
echo -n "ab/cur5.so C3: " >> gpurun_out/ab18.log; PLSSVM_LIB_PATH=$L/ab/cur5.so timeout 120 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 400 >> gpurun_out/ab18.log 2>&1

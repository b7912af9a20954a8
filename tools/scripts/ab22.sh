# A/B: fp64 2 slabs/stage (pass 0: 2 or 3 slabs), fp32 4 vs 5 slabs/stage (2 stages); tests on the variants
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
PLSSVM_LIB_PATH=$L/ab/f64s2p3.so timeout 900 python -m pytest tests/test_gpu_fp64_engines.py -x -q > gpurun_out/ab22_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab22_tests.log
PLSSVM_LIB_PATH=$L/ab/s5st2.so timeout 900 python -m pytest tests/test_gpu_fp32_ozaki.py -x -q >> gpurun_out/ab22_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab22_tests.log
for i in 1 2 3; do for v in ab/f64s2.so ab/f64s2p3.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1000
done; for v in ab/s4st2b.so ab/s5st2.so; do
  echo -n "$v C3: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 400
done; done > gpurun_out/ab22.log 2>&1

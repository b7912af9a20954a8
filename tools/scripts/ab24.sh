# A/B after the large stages: 16 epilogue warps (EPI=16) vs 8; C1 products, C3; fp64 tests on the variant
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
PLSSVM_LIB_PATH=$L/ab/epi16.so timeout 900 python -m pytest tests/test_gpu_fp64_engines.py -x -q > gpurun_out/ab24_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab24_tests.log
for i in 1 2 3; do for v in ab/big.so ab/epi16.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1000
  echo -n "$v C3: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 400
done; done > gpurun_out/ab24.log 2>&1

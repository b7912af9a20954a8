# A/B: pass-0 drain reads levels 0-2 before the release, level 3 after it (under pass 1's MMAs) vs
# the previous build; C1 bench loop, C2 standalone product; then the implicit-product GPU tests.
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
PLSSVM_DEBUG=1 timeout 100 python tools/run_matvec.py --config C1 --synth --repeats 2 > gpurun_out/ab9_debug.log 2>&1
for i in 1 2 3; do for v in ab/pair.so ab/drain3.so; do
  PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/ab_step.py C1 15
done; done > gpurun_out/ab9.log 2>&1
for v in ab/pair.so ab/drain3.so; do
  echo -n "$v C2: "; PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/run_matvec.py --config C2 --synth --repeats 10
done >> gpurun_out/ab9.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp64_engines.py tests/test_gpu_cg_graph.py -x -q > gpurun_out/ab9_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab9_tests.log

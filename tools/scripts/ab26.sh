# A/B: low-rank product with <x_{m-1}, t> computed once (k_lastdot) vs per row-dot warp; C2 low-rank
# products; the low-rank / linear tests on the new build
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
PLSSVM_LIB_PATH=$L/ab/lr_new.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_cg_graph.py -x -q -k "lowrank or linear or graph" > gpurun_out/ab26_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab26_tests.log
for i in 1 2 3; do for v in ab/lr_old.so ab/lr_new.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/run_matvec.py --config C2 --synth --mode lowrank --repeats 200
done; done > gpurun_out/ab26.log 2>&1

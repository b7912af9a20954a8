# A/B: one-GPU product pair-tiles with no dropped half (oz_pair_tiles_matvec) vs HEAD, bench loop (C1),
# then the GPU tests that exercise the implicit int8 product.
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
for i in 1 2 3; do for v in ab/head.so ab/pair.so; do
  PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/ab_step.py C1 15
done; done > gpurun_out/ab8.log 2>&1
for v in ab/head.so ab/pair.so; do
  echo -n "$v C3: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 400
  echo -n "$v C2: "; PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/run_matvec.py --config C2 --synth --repeats 10
done >> gpurun_out/ab8.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp64_engines.py tests/test_gpu_fp32_ozaki.py tests/test_gpu_cg_graph.py tests/test_gpu_cg_variants.py -x -q > gpurun_out/ab8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab8_tests.log

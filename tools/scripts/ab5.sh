# A/B: 8 vs 16 epilogue warps in k_tile_ozaki (C1 fp64 RBF, C3 fp32 poly), sustained products + parity spot check
L=paper_2202_12674_b200/lib
echo -n "epi16 smoke: "; PLSSVM_LIB_PATH=$L/ab/epi16.so timeout 60 python tools/run_matvec.py --config C1 --synth --repeats 3 --compare > gpurun_out/ab5.log 2>&1 || { echo "epi16 failed/hung" >> gpurun_out/ab5.log; exit 0; }
for i in 1 2; do for v in ab/epi8.so ab/epi16.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 60 python tools/run_matvec.py --config C1 --synth --repeats 1000 --compare
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 60 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 600
done; done >> gpurun_out/ab5.log 2>&1
PLSSVM_LIB_PATH=$L/ab/epi16.so timeout 400 python -m pytest tests/test_gpu_fp64_engines.py tests/test_gpu_fp32_ozaki.py -x -q >> gpurun_out/ab5.log 2>&1

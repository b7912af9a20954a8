# fp32 int8 engine: early TMEM release (drain = level combination only) -- parity, A/B vs the round-2 start, cycle accounting
timeout 900 python -m pytest tests/test_gpu_fp32_ozaki.py tests/test_gpu_fp64_engines.py -x -q > gpurun_out/ab3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab3_tests.log
L=paper_2202_12674_b200/lib
for i in 1 2; do for v in ab/head.so libplssvm_b200.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 600
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1000
done; done > gpurun_out/ab3.log 2>&1
PLSSVM_EXPERIMENT_LIB=1 timeout 200 python tools/oz_profile.py C3 10 >> gpurun_out/ab3.log 2>&1

# A/B: fp64 pass order -- V pass (levels 0-3) first [wlast, default] vs W pass (levels 4-6, 18 pairs) first [wfirst]
L=paper_2202_12674_b200/lib
echo -n "wfirst smoke: "; PLSSVM_LIB_PATH=$L/ab/wfirst.so timeout 60 python tools/run_matvec.py --config C1 --synth --repeats 3 --compare > gpurun_out/ab6.log 2>&1 || { echo "wfirst failed/hung" >> gpurun_out/ab6.log; exit 0; }
for i in 1 2; do for v in ab/wlast.so ab/wfirst.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 60 python tools/run_matvec.py --config C1 --synth --repeats 1000 --compare
done; done >> gpurun_out/ab6.log 2>&1
for v in ab/wlast.so ab/wfirst.so; do echo -n "$v C2: "; PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/run_matvec.py --config C2 --synth --repeats 12; done >> gpurun_out/ab6.log 2>&1
PLSSVM_LIB_PATH=$L/ab/wfirst.so timeout 400 python -m pytest tests/test_gpu_fp64_engines.py -x -q >> gpurun_out/ab6.log 2>&1

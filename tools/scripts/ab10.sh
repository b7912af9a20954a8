# A/B: suspend-time hint on the TMA producer's and the epilogue's mbarrier waits (PLSSVM_OZ_SLEEP=20000 ns)
# vs the current build (drain3.so) -- does spinning cost power at the 1 kW cap?
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
for i in 1 2 3; do for v in ab/drain3.so ab/sleep.so; do
  PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/ab_step.py C1 15
done; done > gpurun_out/ab10.log 2>&1
for v in ab/drain3.so ab/sleep.so; do
  echo -n "$v C3: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 400
done >> gpurun_out/ab10.log 2>&1

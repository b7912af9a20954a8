# Experiment: does epilogue instruction work cost time at the power cap?  tax.so evaluates a second
# exp per Q~ entry (-DPLSSVM_OZ_EPI_TAX, ~+12 DP/int instructions per entry) vs the current build.
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
for i in 1 2 3; do for v in ab/cur.so ab/tax.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1000
done; done > gpurun_out/ab11.log 2>&1
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv >> gpurun_out/ab11.log 2>&1

# bench loop (product + predict) with the large stages (big.so) vs the previous stage setup (cur6.so)
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
for i in 1 2; do for v in ab/cur6.so ab/big.so; do
  PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/ab_step.py C1 12
done; done > gpurun_out/ab23.log 2>&1

# A/B of epilogue variants (sustained, back-to-back C1 products); libs under paper_2202_12674_b200/lib/ab
L=paper_2202_12674_b200/lib
for i in 1 2; do
for v in ab/head.so libplssvm_b200.so ab/conv_exp64.so ab/conv_exp64_shift.so ab/conv_exp256_shift.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1500
done
done

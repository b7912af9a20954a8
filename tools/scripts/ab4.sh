# A/B: pipeline depth of k_tile_ozaki (fp64 4 -> 5 stages, fp32 8 -> 10), C1 / C3 sustained products
L=paper_2202_12674_b200/lib
for i in 1 2; do for v in ab/head2.so ab/st5_10.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1000
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 600
done; done > gpurun_out/ab4.log 2>&1

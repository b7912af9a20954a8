# A/B: fp32 int8 engine with 2 slabs (64 features) per pipeline stage (4 or 5 stages of 36 KiB) vs 1 slab
# (8 stages of 18 KiB); C3 products, then the fp32 engine tests on the variant.
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
PLSSVM_LIB_PATH=$L/ab/slabs2.so timeout 900 python -m pytest tests/test_gpu_fp32_ozaki.py -x -q > gpurun_out/ab17_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab17_tests.log
for i in 1 2 3; do for v in ab/cur4.so ab/slabs2.so ab/slabs2s5.so; do
  echo -n "$v C3: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 400
done; done > gpurun_out/ab17.log 2>&1

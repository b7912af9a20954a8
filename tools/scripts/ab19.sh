# A/B: fp32 engine slabs per stage / stage count: cur5 (2 slabs, 4 stages), s2st3, s3st3, s4st3; C3 products;
# fp32 tests on the 3- and 4-slab variants (3 slabs: nk = 64 is not a multiple, the last stage is partial)
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
for v in s3st3 s4st3; do PLSSVM_LIB_PATH=$L/ab/$v.so timeout 900 python -m pytest tests/test_gpu_fp32_ozaki.py -x -q > gpurun_out/ab19_tests_$v.log 2>&1; echo "rc=$?" >> gpurun_out/ab19_tests_$v.log; done
for i in 1 2 3; do for v in ab/cur5.so ab/s2st3.so ab/s3st3.so ab/s4st3.so; do
  echo -n "$v C3: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 400
done; done > gpurun_out/ab19.log 2>&1

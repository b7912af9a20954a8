# A/B: what makes the large stages faster -- the MMA-side wait + tcgen05 fence per stage, or the stage
# handshake itself?  big (2 slabs x 2 stages), fg1s4 (1 slab x 4 stages, fence per slab), fg2 (1 slab x 4
# stages, full-barrier waits and ONE fence per 2 slabs, commits per slab: earlier refills)
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
PLSSVM_LIB_PATH=$L/ab/fg2.so timeout 900 python -m pytest tests/test_gpu_fp64_engines.py -x -q > gpurun_out/ab25_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab25_tests.log
for i in 1 2 3; do for v in ab/big.so ab/fg1s4.so ab/fg2.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1000
done; done > gpurun_out/ab25.log 2>&1

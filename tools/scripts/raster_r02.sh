# One digit layout for both operand roles: parity, then the L2 raster group size at C1 / C3
# (experiment build: PLSSVM_OZ_GROUP), time and DRAM bytes per product.
timeout 900 python -m pytest tests/test_gpu_fp64_engines.py tests/test_gpu_fp32_ozaki.py tests/test_gpu_parity.py -x -q > gpurun_out/r_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r_tests.log
for c in "C1 0" "C3 2"; do set -- $c
  for G in 0 32 64 96; do
    echo "== $1 G=$G"
    PLSSVM_EXPERIMENT_LIB=1 PLSSVM_OZ_GROUP=$G timeout 120 python tools/run_matvec.py --config $1 --synth --fp32-engine $2 --repeats 300
    PLSSVM_EXPERIMENT_LIB=1 PLSSVM_OZ_GROUP=$G timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:k_tile_ozaki -s 2 -c 1 python tools/run_matvec.py --config $1 --synth --fp32-engine $2 --repeats 3 2>&1 | grep -E "dram__bytes|gpu__time"
  done
done > gpurun_out/r_raster.log 2>&1

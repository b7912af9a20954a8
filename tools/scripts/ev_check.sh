# after double-buffered CG timing events: loop / variant / parity / multi-rank tests, probe, bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_cg_graph.py tests/test_gpu_cg_variants.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_num_gpus.py -x -q > gpurun_out/e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/e_tests.log
timeout 300 python tools/overhead_probe.py C1 6 > gpurun_out/e_probe.log 2>&1
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/e_bench.log 2>&1

timeout 900 python -m pytest tests/test_gpu_cg_graph.py tests/test_gpu_cg_variants.py tests/test_gpu_multirank.py tests/test_gpu_num_gpus.py -x -q > gpurun_out/t11.log 2>&1; echo "rc=$?" >> gpurun_out/t11.log
timeout 200 python tools/overhead_probe.py C1 8 > gpurun_out/ov11.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b11.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_cg_fused --csv --log-file gpurun_out/l11.csv python tools/ab_step.py C1 1 > /dev/null 2>&1

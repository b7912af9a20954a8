SEL64='test_engines_match_oracle and (130-31) and 0-1'
timeout 900 compute-sanitizer --tool racecheck --print-limit 40 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fp64_engines.py -k "$SEL64" > gpurun_out/race64.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 40 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_cg_graph.py -k "test_fused_vector_kernel_bit_identical and 1000-33 and 1-" > gpurun_out/racecg.log 2>&1

# compute-sanitizer over small GPU parity cases (run under gpurun from the repo root).
# Both fp64 engines (Ozaki kernel in MATVEC / PRECOMPUTE / PREDICT x 3 kernels, DMMA), the table
# exp range test, the CUDA-graph CG loop.  Output: gpurun_out/sanitize.log
SEL='test_engines_match_oracle and (130-31 or 257-33) or table_exp and (0.3 or 40.0) or test_graph_loop_bit_identical and (256-16 or 777-20)'
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x -p no:cacheprovider \
      tests/test_gpu_fp64_engines.py tests/test_gpu_cg_graph.py -k "$SEL" 2>&1 | grep -vE "^\s*$" | tail -25
done

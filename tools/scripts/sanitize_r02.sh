# compute-sanitizer over the round-2 kernels (gpurun, repo root): the one-layout int8 engines (both roles
# from one digit array, fp64 and fp32, MATVEC / PRECOMPUTE / PREDICT), the raw-X split with padding rows,
# k_row_peak validation, the exponent-range rule, k_cg_fused (cooperative, grid barriers) in both loops.
SEL64='test_engines_match_oracle and (130-31 or 257-33) or table_exp and (0.3) or exponent_range'
SEL32='(test_fp32_ozaki_product_matches_oracle and (257-33 or 1000-33)) or test_fp32_ozaki_predict_and_train'
SELCG='test_fused_vector_kernel_bit_identical'
for tool in memcheck racecheck initcheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x -p no:cacheprovider \
      tests/test_gpu_fp64_engines.py -k "$SEL64" 2>&1 | grep -vE "^\s*$" | tail -8
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x -p no:cacheprovider \
      tests/test_gpu_fp32_ozaki.py -k "$SEL32" 2>&1 | grep -vE "^\s*$" | tail -8
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x -p no:cacheprovider \
      tests/test_gpu_cg_graph.py -k "$SELCG" 2>&1 | grep -vE "^\s*$" | tail -8
done

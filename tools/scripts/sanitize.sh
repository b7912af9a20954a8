# compute-sanitizer over small GPU parity cases (both fp64 engines incl. the 2-SM Ozaki kernel)
SEL='tests/test_gpu_fp64_engines.py -k "engines_match_oracle and (130-31 or 257-33 or 384-64) or zero_rows or integer or train_and_predict"'
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  eval timeout 900 compute-sanitizer --tool $tool --target-processes all python -m pytest $SEL -q -p no:cacheprovider 2>&1 | grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Error|hazard" | head -20
done

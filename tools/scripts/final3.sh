# After the large-stage change: every GPU test, smoke, the bench line, the launch list, ncu of the C1 / C3
# products, the per-config sweep.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/h_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/h_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/h_smoke.log
bash tools/scripts/profile_final.sh

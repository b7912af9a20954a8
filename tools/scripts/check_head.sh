# Full GPU check of HEAD (gpurun, repo root): every GPU test, smoke(), the default bench line.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/h_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/h_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/h_smoke.log
timeout 600 python bench.py > gpurun_out/h_bench.log 2>&1; echo "rc=$?" >> gpurun_out/h_bench.log

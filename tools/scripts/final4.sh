# Last checks of the round: every GPU test + smoke on the final build, and the multi-rank bench path
# (2 ranks on one GPU through the host-staged gloo transport: a logic check, not a measurement)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/z_tests.log 2>&1; echo "rc=$?" >> gpurun_out/z_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/z_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/z_smoke.log
timeout 900 python bench.py --gpus 2 --transport gloo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/z_mr.log 2>&1; echo "rc=$?" >> gpurun_out/z_mr.log

# Full GPU suite + host overhead probe + bench after the library-stream change (one stream per thread and
# device instead of one per call; torch's default stream passed as cudaStreamLegacy).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s_smoke.log
timeout 300 python tools/host_overhead.py C1 4 > gpurun_out/s_hov.log 2>&1
timeout 300 python tools/overhead_probe.py C1 6 > gpurun_out/s_probe.log 2>&1
timeout 600 python bench.py > gpurun_out/s_bench.log 2>&1; echo "rc=$?" >> gpurun_out/s_bench.log

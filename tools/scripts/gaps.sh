# Where the non-product time of a C1 bench step goes (gpurun, repo root): kernel timeline with gaps,
# the overhead probe with and without a concurrent nvidia-smi -lms 200 sampler (bench.py's clocks line).
mkdir -p gpurun_out
timeout 300 python tools/timeline.py C1 3 > gpurun_out/g_timeline.log 2>&1
timeout 300 python tools/overhead_probe.py C1 8 > gpurun_out/g_probe_nosmi.log 2>&1
nvidia-smi --id=0 --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 200 > /dev/null 2>&1 &
SMI=$!
timeout 300 python tools/overhead_probe.py C1 8 > gpurun_out/g_probe_smi.log 2>&1
kill $SMI

nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 100 > gpurun_out/clk10.csv &
SMI=$!
for f in 0 8 0 8 1 3 5; do PLSSVM_OZ_DEBUG=$f timeout 300 python tools/run_matvec.py --config C2 --repeats 4 | sed "s/^/dbg=$f /"; sleep 1; done
kill $SMI

nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/clk_c2.csv &
SMI=$!
timeout 300 python tools/run_matvec.py --config C2 --repeats 8
PLSSVM_OZ_DEBUG=3 timeout 300 python tools/run_matvec.py --config C2 --repeats 8
kill $SMI
timeout 300 python tools/run_matvec.py --config C2 --repeats 2 --fp64-engine 1

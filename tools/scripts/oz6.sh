for f in 0 1 3 5; do PLSSVM_OZ_DEBUG=$f timeout 300 python tools/run_matvec.py --config C2 --repeats 2 | sed "s/^/dbg=$f /"; done
for f in 0 1 3 5; do PLSSVM_OZ_DEBUG=$f timeout 300 python tools/run_matvec.py --config C1 --repeats 3 | sed "s/^/dbg=$f /"; done

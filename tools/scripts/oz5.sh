timeout 120 python tools/run_matvec.py --config C0 --compare --repeats 2
timeout 120 python tools/run_matvec.py --config C1 --m 1000 --d 100 --compare --repeats 2
timeout 120 python tools/run_matvec.py --config C1 --m 1000 --d 100 --kernel 0 --compare --repeats 2
timeout 120 python tools/run_matvec.py --config C1 --m 1000 --d 100 --kernel 1 --compare --repeats 2
timeout 180 python tools/run_matvec.py --config C1 --compare --repeats 5
timeout 300 python tools/run_matvec.py --config C2 --compare --repeats 2
for f in 1 5; do PLSSVM_OZ_DEBUG=$f timeout 300 python tools/run_matvec.py --config C2 --repeats 2 | sed "s/^/dbg=$f /"; done

PLSSVM_OZ_DEBUG=1 timeout 180 python tools/run_matvec.py --config C1 --repeats 5
PLSSVM_OZ_DEBUG=3 timeout 180 python tools/run_matvec.py --config C1 --repeats 5
PLSSVM_OZ_DEBUG=2 timeout 180 python tools/run_matvec.py --config C1 --repeats 5
PLSSVM_OZ_DEBUG=3 timeout 300 python tools/run_matvec.py --config C2 --repeats 2

timeout 60 python tools/run_matvec.py --config C0 --compare --repeats 2
timeout 60 python tools/run_matvec.py --config C1 --m 1000 --d 100 --compare --repeats 2
timeout 120 python tools/run_matvec.py --config C1 --compare --repeats 5
timeout 300 python tools/run_matvec.py --config C2 --compare --repeats 3
timeout 600 python -m pytest tests/test_gpu_fp64_engines.py -q -x 2>&1 | tail -3

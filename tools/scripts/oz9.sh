timeout 120 python tools/run_matvec.py --config C1 --m 1000 --d 100 --compare --repeats 2
timeout 180 python tools/run_matvec.py --config C1 --compare --repeats 5
timeout 300 python tools/run_matvec.py --config C2 --compare --repeats 2
timeout 600 python bench.py > gpurun_out/bench_oz7.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_oz7.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_ozaki -s 2 -c 1 -o gpurun_out/ncu_oz7_c1 python tools/run_matvec.py --config C1 --repeats 3 > /dev/null 2>&1

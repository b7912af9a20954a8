timeout 180 python tools/run_matvec.py --config C1 --compare --repeats 5
timeout 120 python tools/run_matvec.py --config C1 --m 1000 --d 100 --compare --repeats 2
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tile_ozaki -s 1 -c 1 -o gpurun_out/oz_c1b python tools/run_matvec.py --config C1 --repeats 2 > /dev/null 2>&1
ncu -i gpurun_out/oz_c1b.ncu-rep --page raw --csv > gpurun_out/oz_c1b_raw.csv 2>/dev/null
ncu -i gpurun_out/oz_c1b.ncu-rep --page source --csv > gpurun_out/oz_c1b_src.csv 2>/dev/null

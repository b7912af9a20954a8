# One-GPU evidence pass (run under gpurun from the repo root): GPU tests, bench line, launch list
# of two bench steps, ncu --set full of the dominant kernel at C1 (bench data), sanitizer smoke.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_ozaki -s 2 -c 1 -f \
    -o gpurun_out/ncu_oz_c1 python tools/run_matvec.py --config C1 --synth --repeats 3 > /dev/null 2>&1

# Round-2 final evidence pass (gpurun, repo root): bench line, launch list of two bench steps, ncu --set full
# of the C1 product (fp64 int8 engine) and the C3 product (fp32 int8 engine), per-config sweep.
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/f_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_c1.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
cap() {  # name, ncu args...
    local n=$1; shift
    timeout 900 ncu --set full --clock-control none --import-source on -f -o /tmp/$n "$@" > /dev/null 2>&1
    python tools/ncu_summary.py /tmp/$n.ncu-rep > gpurun_out/$n.summary.txt 2>&1
    ncu -i /tmp/$n.ncu-rep --page details > gpurun_out/$n.details.txt 2>/dev/null
}
cap f_ncu_oz_c1 -k regex:k_tile_ozaki -s 2 -c 1 python tools/run_matvec.py --config C1 --synth --repeats 3
cap f_ncu_oz32_c3 -k regex:k_tile_ozaki -s 2 -c 1 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 3
timeout 1500 python tools/sweep.py --out gpurun_out/f_sweep.jsonl > gpurun_out/f_sweep.log 2>&1
du -sh gpurun_out

# Round-2 evidence pass (gpurun, repo root): CG tests, bench, launch list of two bench steps, ncu --set full
# of the dominant kernel (C1), of the fused CG vector kernel and of the fp32 int8 engine at C3.
# Reports are reduced on the box (raw page CSV + a summary) so gpurun_out stays under its 64 MiB cap.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cg_graph.py tests/test_gpu_cg_variants.py tests/test_gpu_parity.py -x -q > gpurun_out/p_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p_tests.log
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/p_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches_c1.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
cap() {  # name, ncu args...
    local n=$1; shift
    timeout 900 ncu --set full --clock-control none --import-source on -f -o /tmp/$n "$@" > /dev/null 2>&1
    ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/$n.raw.csv 2>/dev/null
    python tools/ncu_summary.py /tmp/$n.ncu-rep > gpurun_out/$n.summary.txt 2>&1
    ncu -i /tmp/$n.ncu-rep --page details > gpurun_out/$n.details.txt 2>/dev/null
}
cap p_ncu_oz_c1 -k regex:k_tile_ozaki -s 2 -c 1 python tools/run_matvec.py --config C1 --synth --repeats 3
cap p_ncu_cgfused_c1 --cache-control none -k regex:k_cg_fused -s 10 -c 1 python tools/ab_step.py C1 1
cap p_ncu_oz32_c3 -k regex:k_tile_ozaki -s 2 -c 1 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 3
for i in 1 2; do timeout 120 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 200; done > gpurun_out/p_c3.log 2>&1
du -sh gpurun_out

# Round-2 evidence (gpurun, repo root): C2 stagnation test, ncu --set full of the final k_tile_ozaki (C1 fp64,
# C3 fp32), the multi-rank bench spawn path as a dry run (2 ranks on one GPU, host-staged gloo transport:
# NCCL refuses two ranks on one device), and the per-config sweep.  Reports reduced on the box (64 MiB cap).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "stagnation" -x -q -s > gpurun_out/e_stag.log 2>&1; echo "rc=$?" >> gpurun_out/e_stag.log
cap() {
    local n=$1; shift
    timeout 900 ncu --set full --clock-control none --import-source on -f -o /tmp/$n "$@" > /dev/null 2>&1
    python tools/ncu_summary.py /tmp/$n.ncu-rep > gpurun_out/$n.summary.txt 2>&1
    ncu -i /tmp/$n.ncu-rep --page details > gpurun_out/$n.details.txt 2>/dev/null
}
cap e_ncu_oz_c1 -k regex:k_tile_ozaki -s 2 -c 1 python tools/run_matvec.py --config C1 --synth --repeats 3
cap e_ncu_oz32_c3 -k regex:k_tile_ozaki -s 2 -c 1 python tools/run_matvec.py --config C3 --synth --fp32-engine 2 --repeats 3
timeout 600 python bench.py --gpus 2 --transport gloo --steps 3 --warmup 3 > gpurun_out/e_bench_gloo2.log 2>&1; echo "rc=$?" >> gpurun_out/e_bench_gloo2.log
timeout 2400 python tools/sweep.py --out gpurun_out/e_sweep.jsonl > gpurun_out/e_sweep.log 2>&1
du -sh gpurun_out

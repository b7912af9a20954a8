# low-rank (NEXT-2) product kernels: parity tests, then A/B vs the previous kernels at C2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cg_graph.py tests/test_gpu_multirank.py -x -q -k "lowrank or LOWRANK or c2_full_training or ridge or linear or graph_loop_bit or fused or row_sharded" > gpurun_out/ab7_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab7_tests.log
L=paper_2202_12674_b200/lib
for i in 1 2; do for v in ab/head2.so libplssvm_b200.so; do
  echo -n "$v: "; PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/run_matvec.py --config C2 --synth --mode lowrank --repeats 200
done; done > gpurun_out/ab7.log 2>&1

# e2e (host buffers) probe: per-call library stream (cur2.so) vs the cached per-thread stream (stream.so)
L=paper_2202_12674_b200/lib
mkdir -p gpurun_out
for v in ab/cur2.so ab/stream.so ab/cur2.so ab/stream.so; do
  echo "== $v"; PLSSVM_LIB_PATH=$L/$v timeout 200 python tools/e2e_probe.py C1
done > gpurun_out/ab15.log 2>&1

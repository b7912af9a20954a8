set -x
H=paper_2202_12674_b200/lib/ab/head.so
N=paper_2202_12674_b200/lib/libplssvm_b200.so
for i in 1 2; do
PLSSVM_LIB_PATH=$H timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1500
PLSSVM_LIB_PATH=$N timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1500
done
PLSSVM_EXPERIMENT_LIB=1 PLSSVM_OZ_DEBUG=1 timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1500
PLSSVM_EXPERIMENT_LIB=1 PLSSVM_OZ_DEBUG=4 timeout 120 python tools/run_matvec.py --config C1 --synth --repeats 1500
for i in 1 2 3; do
PLSSVM_LIB_PATH=$H timeout 120 python tools/ab_step.py C1 12
PLSSVM_LIB_PATH=$N timeout 120 python tools/ab_step.py C1 12
done

"""B200-native PLSSVM hot path: LS-SVM training by CG on the reduced kernel system Q~
(arXiv 2202.12674) behind the C ABI include/plssvm.h.  This package holds the CUDA sources
(csrc/), the in-tree build (_build.py) and the thin ctypes binding (binding.py).
It never imports ``oracle/``; it has no CPU fallback."""
from .binding import (  # noqa: F401
    LINEAR, POLYNOMIAL, RBF, F64, F32, MODE_AUTO, MODE_IMPLICIT, MODE_CACHED, MODE_LOWRANK, FP64_AUTO, FP64_OZAKI, FP64_DMMA, CG_AUTO, CG_BATCHED, CG_GRAPH,
    MULTI_GPU_ROWS, MULTI_GPU_FEATURES, CG_SHEWCHUK, CG_SINGLE_REDUCTION, FP32_TCGEN05,
    FP32_FFMA, FP32_OZAKI, FP32_AUTO, TRANSPORT_AUTO, TRANSPORT_NCCL, TRANSPORT_PEER, STOP_CONVERGED, STOP_MAX_ITER,
    STOP_FIXED, STOP_STAGNATED, STOP_BREAKDOWN, OK, E_INVALID_ARG, E_LABELS, E_OOM, E_CUDA, E_NCCL, E_NUMERICAL,
    W_NOT_CONVERGED, E_IO, PlssvmError, options, load,
    plssvm_train, plssvm_train_ex, plssvm_predict, plssvm_predict_ex, plssvm_qtilde_matvec, plssvm_partition,
    plssvm_feature_partition,
    plssvm_version, plssvm_device_count, plssvm_last_error, plssvm_comm_unique_id, plssvm_comm_init,
    plssvm_comm_destroy, plssvm_comm_init_callbacks, comm_from_torch_distributed, comm_host_staged,
    plssvm_libsvm_read, plssvm_libsvm_write, plssvm_model_write, plssvm_model_read, plssvm_scale_fit,
    plssvm_scale_apply, cli_path,
)

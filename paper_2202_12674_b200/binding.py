"""Thin ctypes binding of include/plssvm.h (argument marshalling only).

Every function here has the name of the C entry point it calls.  Host inputs are numpy
arrays; torch CUDA tensors are passed as device pointers (options.device_pointers = 1) on
torch's current stream.  No arithmetic of the method happens in Python, and there is no
fallback: if the shared library is missing or the call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

from . import _build

LINEAR, POLYNOMIAL, RBF = 0, 1, 2
F64, F32 = 0, 1
MODE_AUTO, MODE_IMPLICIT, MODE_CACHED, MODE_LOWRANK = 0, 1, 2, 3
FP64_AUTO, FP64_OZAKI, FP64_DMMA = 0, 1, 2
CG_AUTO, CG_BATCHED, CG_GRAPH = 0, 1, 2
MULTI_GPU_ROWS, MULTI_GPU_FEATURES = 0, 1
CG_SHEWCHUK, CG_SINGLE_REDUCTION = 0, 1
FP32_TCGEN05, FP32_FFMA, FP32_OZAKI, FP32_AUTO = 0, 1, 2, 3
TRANSPORT_AUTO, TRANSPORT_NCCL, TRANSPORT_PEER = 0, 1, 2
CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy
STOP_CONVERGED, STOP_MAX_ITER, STOP_FIXED, STOP_STAGNATED, STOP_BREAKDOWN = 0, 1, 2, 3, 4
OK, E_INVALID_ARG, E_LABELS, E_OOM, E_CUDA, E_NCCL, E_NUMERICAL, W_NOT_CONVERGED, E_IO = range(9)
STATUS_NAMES = {0: "OK", 1: "E_INVALID_ARG", 2: "E_LABELS", 3: "E_OOM", 4: "E_CUDA", 5: "E_NCCL",
                6: "E_NUMERICAL", 7: "W_NOT_CONVERGED", 8: "E_IO"}

EXPORTS = ["plssvm_default_options", "plssvm_train", "plssvm_train_f32", "plssvm_train_ex", "plssvm_predict",
           "plssvm_predict_f32", "plssvm_predict_ex", "plssvm_qtilde_matvec", "plssvm_comm_unique_id",
           "plssvm_comm_init", "plssvm_comm_init_callbacks", "plssvm_comm_destroy", "plssvm_partition",
           "plssvm_feature_partition", "plssvm_last_error", "plssvm_version", "plssvm_device_count",
           "plssvm_libsvm_read", "plssvm_libsvm_write", "plssvm_model_write", "plssvm_model_read", "plssvm_scale_fit",
           "plssvm_scale_apply"]


class plssvm_options_t(ct.Structure):
    _fields_ = [("mode", ct.c_int32), ("x0", ct.c_int32), ("max_iter", ct.c_int64), ("replace_every", ct.c_int64),
                ("fixed_iter", ct.c_int64), ("device", ct.c_int32), ("device_pointers", ct.c_int32),
                ("stream", ct.c_void_p), ("comm", ct.c_void_p), ("cache_budget_bytes", ct.c_int64),
                ("fp32_engine", ct.c_int32), ("linear_w", ct.c_int32), ("fp64_engine", ct.c_int32),
                ("cg_loop", ct.c_int32), ("multi_gpu", ct.c_int32), ("cg_variant", ct.c_int32),
                ("num_gpus", ct.c_int32), ("transport", ct.c_int32), ("true_residual", ct.c_int32),
                ("reserved0", ct.c_int32), ("residual_trace", ct.c_void_p), ("residual_trace_len", ct.c_int64)]


class plssvm_stats_t(ct.Structure):
    _fields_ = [("iterations", ct.c_int64), ("matvecs", ct.c_int64), ("rel_residual", ct.c_double),
                ("mode_used", ct.c_int32), ("num_ranks", ct.c_int32), ("t_h2d", ct.c_double),
                ("t_transform", ct.c_double), ("t_q", ct.c_double), ("t_alloc", ct.c_double),
                ("t_precompute", ct.c_double),
                ("t_cg", ct.c_double), ("t_bias_d2h", ct.c_double), ("t_total", ct.c_double),
                ("t_matvec", ct.c_double), ("t_matvec_min", ct.c_double), ("bytes_per_gpu", ct.c_int64),
                ("gpu_launches", ct.c_int64), ("launches_in_cg", ct.c_int64), ("fp64_engine_used", ct.c_int32),
                ("cg_loop_used", ct.c_int32), ("fp32_engine_used", ct.c_int32), ("allgather_fused", ct.c_int32),
                ("t_comm", ct.c_double), ("rel_residual_true", ct.c_double), ("stop_reason", ct.c_int32),
                ("transport_used", ct.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


ALLREDUCE_CB = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.c_void_p, ct.c_int64, ct.c_void_p)
ALLGATHER_CB = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.c_void_p, ct.c_int64, ct.c_int32, ct.c_void_p)
REDUCE_SCATTER_CB = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_int64, ct.c_int32, ct.c_void_p)


class plssvm_comm_callbacks_t(ct.Structure):
    _fields_ = [("ctx", ct.c_void_p), ("allreduce_sum_f64", ALLREDUCE_CB), ("allgather", ALLGATHER_CB),
                ("reduce_scatter_sum", REDUCE_SCATTER_CB)]


class PlssvmError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib_path() -> str:
    """The product library; PLSSVM_EXPERIMENT_LIB=1 selects the experiment build (tools/ only: its
    PLSSVM_OZ_DEBUG switches make results wrong; bench.py refuses to run with it)."""
    if os.environ.get("PLSSVM_LIB_PATH"):  # tools/ A/B runs of two builds (bench.py refuses PLSSVM_*)
        return os.environ["PLSSVM_LIB_PATH"]
    return _build.LIB_EXP if os.environ.get("PLSSVM_EXPERIMENT_LIB") == "1" else _build.LIB


def load(build_if_missing: bool = True):
    """Load libplssvm_b200.so (building it in-tree first if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        if not build_if_missing:
            raise FileNotFoundError(f"{path} missing: run __graft_entry__.build()")
        _build.build(variant="exp" if path == _build.LIB_EXP else "product")
    L = ct.CDLL(path)
    vp, i64, i32, d, i = ct.c_void_p, ct.c_int64, ct.c_int32, ct.c_double, ct.c_int
    L.plssvm_default_options.argtypes = [ct.POINTER(plssvm_options_t)]
    L.plssvm_default_options.restype = None
    L.plssvm_train_ex.argtypes = [vp, vp, i64, i64, i, i, d, i, d, d, d, ct.POINTER(plssvm_options_t), vp, vp,
                                  ct.POINTER(plssvm_stats_t)]
    L.plssvm_train.argtypes = [vp, vp, i64, i64, i, d, i, d, d, d, vp, vp]
    L.plssvm_train_f32.argtypes = [vp, vp, i64, i64, i, ct.c_float, i, ct.c_float, ct.c_float, ct.c_float, vp, vp]
    L.plssvm_predict.argtypes = [vp, vp, d, i64, i64, i, d, i, d, vp, i64, vp, vp]
    L.plssvm_predict_f32.argtypes = [vp, vp, ct.c_float, i64, i64, i, ct.c_float, i, ct.c_float, vp, i64, vp, vp]
    L.plssvm_predict_ex.argtypes = [vp, vp, d, i64, i64, i, i, d, i, d, vp, i64, ct.POINTER(plssvm_options_t), vp,
                                    vp, vp]
    L.plssvm_qtilde_matvec.argtypes = [vp, vp, i64, i64, i, i, d, i, d, d, i32, ct.POINTER(plssvm_options_t), vp,
                                       ct.POINTER(ct.c_double)]
    L.plssvm_comm_unique_id.argtypes = [vp]
    L.plssvm_comm_init.argtypes = [vp, i32, i32, i32, ct.POINTER(vp)]
    L.plssvm_comm_destroy.argtypes = [vp]
    L.plssvm_comm_init_callbacks.argtypes = [ct.POINTER(plssvm_comm_callbacks_t), i32, i32, i32, ct.POINTER(vp)]
    L.plssvm_partition.argtypes = [i64, i32, i32, ct.POINTER(i64), ct.POINTER(i64), ct.POINTER(i64)]
    L.plssvm_feature_partition.argtypes = [i64, i32, i32, ct.POINTER(i64), ct.POINTER(i64)]
    pd = ct.POINTER(ct.c_double)
    L.plssvm_libsvm_read.argtypes = [ct.c_char_p, vp, vp, i64, i64, ct.POINTER(i64), ct.POINTER(i64), pd,
                                     ct.POINTER(i32)]
    L.plssvm_libsvm_write.argtypes = [ct.c_char_p, vp, vp, i64, i64]
    L.plssvm_model_write.argtypes = [ct.c_char_p, i, d, i, d, vp, vp, d, i64, i64, vp, pd]
    L.plssvm_model_read.argtypes = [ct.c_char_p, ct.POINTER(i32), pd, ct.POINTER(i32), pd, vp, vp, pd, i64, i64,
                                    ct.POINTER(i64), ct.POINTER(i64), pd]
    L.plssvm_scale_fit.argtypes = [vp, i64, i64, vp, vp]
    L.plssvm_scale_apply.argtypes = [vp, i64, i64, vp, vp, d, d]
    L.plssvm_last_error.restype = ct.c_char_p
    L.plssvm_version.restype = ct.c_char_p
    L.plssvm_device_count.restype = ct.c_int
    for name in EXPORTS:
        if name not in ("plssvm_default_options", "plssvm_last_error", "plssvm_version", "plssvm_device_count"):
            getattr(L, name).restype = ct.c_int
    _lib = L
    return L


def _check(status, allow=(OK,)):
    if status not in allow:
        raise PlssvmError(status, load().plssvm_last_error().decode())
    return status


def _is_torch_cuda(a) -> bool:
    return type(a).__module__.startswith("torch") and getattr(a, "is_cuda", False)


def _dtype_code(a) -> int:
    s = str(a.dtype)
    if s.endswith("float64"):
        return F64
    if s.endswith("float32"):
        return F32
    raise TypeError(f"unsupported dtype {a.dtype}")


def _host(a, dt):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64 if dt == F64 else np.float32))


def options(**kw) -> plssvm_options_t:
    o = plssvm_options_t()
    load().plssvm_default_options(ct.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _same_device_tensor(name, t, X, n):
    """A torch CUDA tensor that can be passed as a device pointer beside X: same dtype, same device,
    contiguous, n elements.  Anything else raises (a wrong dtype would be read with X's element size,
    a host tensor's pointer would be dereferenced on the device)."""
    if not _is_torch_cuda(t):
        raise TypeError(f"{name} must be a CUDA tensor on {X.device} like X (got {type(t).__name__}"
                        f"{' on ' + str(t.device) if hasattr(t, 'device') else ''})")
    if t.device != X.device:
        raise ValueError(f"{name} is on {t.device}, X on {X.device}")
    if t.dtype != X.dtype:
        raise TypeError(f"{name} has dtype {t.dtype}, X has {X.dtype}")
    if t.numel() != n:
        raise ValueError(f"{name} has {t.numel()} elements, expected {n}")
    return t.contiguous()


def _device_opts(o, tensors):
    import torch

    o.device_pointers = 1
    o.device = tensors[0].device.index or 0
    # torch's current stream; its default stream has the handle 0, which the C ABI reads as "no stream"
    # (a library stream, NOT ordered after torch's work on the legacy default stream), so that one is
    # passed as cudaStreamLegacy (0x1)
    o.stream = torch.cuda.current_stream(tensors[0].device).cuda_stream or CUDA_STREAM_LEGACY
    return o


# ------------------------------------------------------------------------------ entry points
def plssvm_version() -> str:
    return load().plssvm_version().decode()


def plssvm_device_count() -> int:
    return load().plssvm_device_count()


def plssvm_last_error() -> str:
    return load().plssvm_last_error().decode()


def plssvm_partition(m: int, nranks: int, rank: int):
    """(row_begin, row_end, m_pad) of `rank` in the padded (m-1)-system (host logic, no GPU)."""
    b, e, mp = ct.c_int64(), ct.c_int64(), ct.c_int64()
    _check(load().plssvm_partition(m, nranks, rank, ct.byref(b), ct.byref(e), ct.byref(mp)))
    return b.value, e.value, mp.value


def plssvm_feature_partition(d: int, nranks: int, rank: int):
    """(f_begin, f_end): the feature slice of `rank` under MULTI_GPU_FEATURES (host logic, no GPU)."""
    b, e = ct.c_int64(), ct.c_int64()
    _check(load().plssvm_feature_partition(d, nranks, rank, ct.byref(b), ct.byref(e)))
    return b.value, e.value


def plssvm_train(X, y, kernel, gamma=1.0, degree=3, coef0=0.0, C=1.0, eps=1e-10):
    """Host numpy in / out, fp64 (plssvm_train) or fp32 (plssvm_train_f32) by X's dtype."""
    dt = F32 if str(getattr(X, "dtype", "")) == "float32" else F64
    X, y = _host(X, dt), _host(y, dt)
    m, d = X.shape
    alpha = np.empty(m, dtype=X.dtype)
    b = np.zeros(1, dtype=X.dtype)
    L = load()
    if dt == F64:
        st = L.plssvm_train(X.ctypes.data, y.ctypes.data, m, d, kernel, gamma, degree, coef0, C, eps,
                            alpha.ctypes.data, b.ctypes.data)
    else:
        st = L.plssvm_train_f32(X.ctypes.data, y.ctypes.data, m, d, kernel, gamma, degree, coef0, C, eps,
                                alpha.ctypes.data, b.ctypes.data)
    _check(st, (OK, W_NOT_CONVERGED))
    return alpha, float(b[0]), st


def plssvm_train_ex(X, y, kernel, gamma=1.0, degree=3, coef0=0.0, C=1.0, eps=1e-10, opts=None, alpha=None, b=None):
    """numpy (host) or torch CUDA tensors (device pointers).  Returns (alpha, b, status, stats)."""
    o = opts if opts is not None else options()
    stats = plssvm_stats_t()
    dt = _dtype_code(X)
    m, d = X.shape
    L = load()
    if _is_torch_cuda(X):
        import torch

        _device_opts(o, [X])
        X = X.contiguous()
        y = _same_device_tensor("y", y, X, m)
        alpha = torch.empty(m, dtype=X.dtype, device=X.device) if alpha is None else alpha
        b = torch.empty(1, dtype=X.dtype, device=X.device) if b is None else b
        if not (alpha.is_contiguous() and b.is_contiguous()):
            raise ValueError("alpha and b outputs must be contiguous")
        alpha, b = _same_device_tensor("alpha", alpha, X, m), _same_device_tensor("b", b, X, 1)
        st = L.plssvm_train_ex(X.data_ptr(), y.data_ptr(), m, d, dt, kernel, gamma, degree, coef0, C, eps,
                               ct.byref(o), alpha.data_ptr(), b.data_ptr(), ct.byref(stats))
        _check(st, (OK, W_NOT_CONVERGED))
        return alpha, b, st, stats
    X, y = _host(X, dt), _host(y, dt)
    alpha = np.empty(m, dtype=X.dtype) if alpha is None else alpha
    b = np.zeros(1, dtype=X.dtype) if b is None else b
    st = L.plssvm_train_ex(X.ctypes.data, y.ctypes.data, m, d, dt, kernel, gamma, degree, coef0, C, eps, ct.byref(o),
                           alpha.ctypes.data, b.ctypes.data, ct.byref(stats))
    _check(st, (OK, W_NOT_CONVERGED))
    return alpha, float(b[0]), st, stats


def plssvm_predict(X, alpha, b, Z, kernel, gamma=1.0, degree=3, coef0=0.0):
    """Host numpy; returns (decision[n], labels[n])."""
    dt = F32 if str(getattr(X, "dtype", "")) == "float32" else F64
    X, alpha, Z = _host(X, dt), _host(alpha, dt), _host(Z, dt)
    m, d = X.shape
    n = Z.shape[0]
    f = np.empty(n, dtype=X.dtype)
    lab = np.empty(n, dtype=np.int32)
    L = load()
    fn = L.plssvm_predict if dt == F64 else L.plssvm_predict_f32
    _check(fn(X.ctypes.data, alpha.ctypes.data, b, m, d, kernel, gamma, degree, coef0, Z.ctypes.data, n,
              f.ctypes.data, lab.ctypes.data))
    return f, lab


def plssvm_predict_ex(X, alpha, b, Z, kernel, gamma=1.0, degree=3, coef0=0.0, opts=None):
    """numpy or torch CUDA tensors.  Returns (decision, labels, (kernel_seconds, launches))."""
    o = opts if opts is not None else options()
    dt = _dtype_code(X)
    m, d = X.shape
    n = Z.shape[0]
    tk = (ct.c_double * 2)()
    L = load()
    if _is_torch_cuda(X):
        import torch

        _device_opts(o, [X])
        X = X.contiguous()
        alpha = _same_device_tensor("alpha", alpha, X, m)
        Z = _same_device_tensor("Z", Z, X, n * d)
        f = torch.empty(n, dtype=X.dtype, device=X.device)
        lab = torch.empty(n, dtype=torch.int32, device=X.device)
        _check(L.plssvm_predict_ex(X.data_ptr(), alpha.data_ptr(), float(b), m, d, dt,
                                   kernel, gamma, degree, coef0, Z.data_ptr(), n, ct.byref(o),
                                   f.data_ptr(), lab.data_ptr(), tk))
        return f, lab, tuple(tk)
    X, alpha, Z = _host(X, dt), _host(alpha, dt), _host(Z, dt)
    f = np.empty(n, dtype=X.dtype)
    lab = np.empty(n, dtype=np.int32)
    _check(L.plssvm_predict_ex(X.ctypes.data, alpha.ctypes.data, float(b), m, d, dt, kernel, gamma, degree, coef0,
                               Z.ctypes.data, n, ct.byref(o), f.ctypes.data, lab.ctypes.data, tk))
    return f, lab, tuple(tk)


def plssvm_qtilde_matvec(X, p, kernel, gamma=1.0, degree=3, coef0=0.0, C=1.0, repeats=1, opts=None):
    """out = Q~ p (length m-1).  Returns (out, (mean_s, min_s, precompute_s))."""
    o = opts if opts is not None else options()
    dt = _dtype_code(X)
    m, d = X.shape
    tk = (ct.c_double * 3)()
    L = load()
    if _is_torch_cuda(X):
        import torch

        _device_opts(o, [X])
        X = X.contiguous()
        p = _same_device_tensor("p", p, X, m - 1)
        out = torch.empty(m - 1, dtype=X.dtype, device=X.device)
        _check(L.plssvm_qtilde_matvec(X.data_ptr(), p.data_ptr(), m, d, dt, kernel, gamma,
                                      degree, coef0, C, repeats, ct.byref(o), out.data_ptr(), tk))
        return out, tuple(tk)
    X, p = _host(X, dt), _host(p, dt)
    out = np.empty(m - 1, dtype=X.dtype)
    _check(L.plssvm_qtilde_matvec(X.ctypes.data, p.ctypes.data, m, d, dt, kernel, gamma, degree, coef0, C, repeats,
                                  ct.byref(o), out.ctypes.data, tk))
    return out, tuple(tk)


def plssvm_comm_unique_id() -> bytes:
    buf = ct.create_string_buffer(128)
    _check(load().plssvm_comm_unique_id(buf))
    return buf.raw


def plssvm_comm_init(uid: bytes, nranks: int, rank: int, device: int):
    h = ct.c_void_p()
    buf = ct.create_string_buffer(uid, 128)
    _check(load().plssvm_comm_init(buf, nranks, rank, device, ct.byref(h)))
    return h.value


_CALLBACK_KEEPALIVE = {}


def plssvm_comm_init_callbacks(allreduce_sum_f64, allgather, nranks: int, rank: int, device: int,
                               reduce_scatter_sum=None):
    """Communicator whose collectives are Python callables (see plssvm.h)."""
    cb = plssvm_comm_callbacks_t(None, ALLREDUCE_CB(allreduce_sum_f64), ALLGATHER_CB(allgather),
                                 REDUCE_SCATTER_CB(reduce_scatter_sum) if reduce_scatter_sum else REDUCE_SCATTER_CB())
    h = ct.c_void_p()
    _check(load().plssvm_comm_init_callbacks(ct.byref(cb), nranks, rank, device, ct.byref(h)))
    _CALLBACK_KEEPALIVE[h.value] = cb
    return h.value


def plssvm_comm_destroy(comm) -> None:
    _check(load().plssvm_comm_destroy(comm))
    _CALLBACK_KEEPALIVE.pop(comm, None)


def comm_host_staged(device: int, circulant: bool = True):
    """Communicator over torch.distributed (any backend, e.g. gloo) with host staging: each
    collective synchronises the driver's stream, copies the device buffer to host, runs the
    torch.distributed collective and copies back.  For testing the row-sharded driver with
    several processes on ONE GPU (NCCL refuses duplicate devices); not a fast path.
    circulant=False omits the reduce-scatter, so implicit mode uses plain row bands."""
    import torch
    import torch.distributed as dist

    cudart = _cudart()
    rank, world = dist.get_rank(), dist.get_world_size()

    def d2h(ptr, nbytes, stream):
        if cudart.cudaStreamSynchronize(ct.c_void_p(stream)) != 0:
            return None
        host = torch.empty(nbytes, dtype=torch.uint8)
        if cudart.cudaMemcpy(ct.c_void_p(host.data_ptr()), ct.c_void_p(ptr), ct.c_size_t(nbytes), 2) != 0:
            return None
        return host

    def h2d(ptr, host):
        # a pageable H2D cudaMemcpy may return before the DMA lands: synchronise the device so
        # the driver's (non-blocking) stream sees the data
        st = cudart.cudaMemcpy(ct.c_void_p(ptr), ct.c_void_p(host.data_ptr()), ct.c_size_t(host.numel()), 1)
        return st or cudart.cudaDeviceSynchronize()

    def allreduce(ctx, buf, count, stream):
        host = d2h(buf, 8 * count, stream)
        if host is None:
            return 1
        t = host.view(torch.float64)
        dist.all_reduce(t)
        return h2d(buf, t.view(torch.uint8))

    def allgather(ctx, buf, count, dtype, stream):
        es = 8 if dtype == F64 else 4
        nb = count * es
        host = d2h(buf + rank * nb, nb, stream)
        if host is None:
            return 1
        parts = [torch.empty(nb, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, host)
        return h2d(buf, torch.cat(parts))

    def reduce_scatter(ctx, send, recv, count, dtype, stream):
        es = 8 if dtype == F64 else 4
        host = d2h(send, world * count * es, stream)
        if host is None:
            return 1
        t = host.view(torch.float64 if dtype == F64 else torch.float32)
        dist.all_reduce(t)  # sum over ranks, then keep this rank's block
        return h2d(recv, t[rank * count:(rank + 1) * count].contiguous().view(torch.uint8))

    return plssvm_comm_init_callbacks(allreduce, allgather, world, rank, device,
                                      reduce_scatter if circulant else None)


_cudart_lib = None


def _cudart():
    global _cudart_lib
    if _cudart_lib is None:
        import glob

        import torch

        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                       "libcudart.so*")) + ["libcudart.so.12", "libcudart.so"]
        for c in cands:
            try:
                _cudart_lib = ct.CDLL(c)
                break
            except OSError:
                continue
        _cudart_lib.cudaMemcpy.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_size_t, ct.c_int]
        _cudart_lib.cudaStreamSynchronize.argtypes = [ct.c_void_p]
    return _cudart_lib


def comm_from_torch_distributed(device: int):
    """Create the NCCL communicator of this rank; torch.distributed only broadcasts the id."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    uid = plssvm_comm_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    if dist.get_backend() == "nccl":
        t = t.cuda(device)
    dist.broadcast(t, 0)
    return plssvm_comm_init(bytes(t.cpu().tolist()), world, rank, device)


# ------------------------------------------------------------------- LIBSVM files (NEXT-4)
def _path(p) -> bytes:
    return os.fsencode(p)


def plssvm_libsvm_read(path, min_d: int = 0):
    """-> (X [m, max(d, min_d)] float64, y_raw [m], labels (distinct, first-seen order))."""
    L = load()
    m, d, nl = ct.c_int64(), ct.c_int64(), ct.c_int32()
    labs = (ct.c_double * 2)()
    _check(L.plssvm_libsvm_read(_path(path), None, None, 0, 0, ct.byref(m), ct.byref(d), labs, ct.byref(nl)))
    D = max(d.value, min_d, 1)
    X = np.zeros((m.value, D))
    y = np.zeros(m.value)
    _check(L.plssvm_libsvm_read(_path(path), X.ctypes.data, y.ctypes.data, m.value, D, ct.byref(m), ct.byref(d), labs,
                                ct.byref(nl)))
    return X, y, [labs[k] for k in range(nl.value)]


def plssvm_libsvm_write(path, X, y):
    X, y = _host(X, F64), _host(y, F64)
    _check(load().plssvm_libsvm_write(_path(path), X.ctypes.data, y.ctypes.data, X.shape[0], X.shape[1]))


def plssvm_model_write(path, kernel, gamma, degree, coef0, X, alpha, b, y, labels):
    X, alpha, y = _host(X, F64), _host(alpha, F64), _host(y, F64)
    labs = (ct.c_double * 2)(float(labels[0]), float(labels[1]))
    _check(load().plssvm_model_write(_path(path), kernel, gamma, degree, coef0, X.ctypes.data, alpha.ctypes.data,
                                     float(b), X.shape[0], X.shape[1], y.ctypes.data, labs))


def plssvm_model_read(path, min_d: int = 0):
    """-> dict(kernel, gamma, degree, coef0, X, alpha, b, labels)."""
    L = load()
    k, dg = ct.c_int32(), ct.c_int32()
    g, r, b = ct.c_double(), ct.c_double(), ct.c_double()
    m, d = ct.c_int64(), ct.c_int64()
    labs = (ct.c_double * 2)()
    args = (ct.byref(k), ct.byref(g), ct.byref(dg), ct.byref(r))
    _check(L.plssvm_model_read(_path(path), *args, None, None, ct.byref(b), 0, 0, ct.byref(m), ct.byref(d), labs))
    D = max(d.value, min_d, 1)
    X = np.zeros((m.value, D))
    alpha = np.zeros(m.value)
    _check(L.plssvm_model_read(_path(path), *args, X.ctypes.data, alpha.ctypes.data, ct.byref(b), m.value, D,
                               ct.byref(m), ct.byref(d), labs))
    return dict(kernel=k.value, gamma=g.value, degree=dg.value, coef0=r.value, X=X, alpha=alpha, b=b.value,
                labels=[labs[0], labs[1]])


def plssvm_scale_fit(X):
    X = _host(X, F64)
    fmin, fmax = np.zeros(X.shape[1]), np.zeros(X.shape[1])
    _check(load().plssvm_scale_fit(X.ctypes.data, X.shape[0], X.shape[1], fmin.ctypes.data, fmax.ctypes.data))
    return fmin, fmax


def plssvm_scale_apply(X, fmin, fmax, lo=-1.0, hi=1.0):
    """Returns a scaled copy (the C call works in place)."""
    X = np.array(X, dtype=np.float64, order="C", copy=True)
    fmin, fmax = _host(fmin, F64), _host(fmax, F64)
    _check(load().plssvm_scale_apply(X.ctypes.data, X.shape[0], X.shape[1], fmin.ctypes.data, fmax.ctypes.data, lo, hi))
    return X


def cli_path() -> str:
    """bin/plssvm (the LIBSVM-style CLI; plssvm-train / -predict / -scale link to it)."""
    return _build.CLI

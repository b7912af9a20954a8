"""CPU-side checks of the C-ABI library: it loads, exports exactly what include/plssvm.h
declares, validates its arguments, implements the host partition rule, and refuses to
compute without a GPU (no CPU fallback)."""
import ctypes as ct
import os
import re

import numpy as np
import pytest

import paper_2202_12674_b200 as pl
from paper_2202_12674_b200 import binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "plssvm.h")).read()
    return sorted(set(re.findall(r"PLSSVM_API\s+[\w\s\*]*?\b(plssvm_\w+)\s*\(", src)))


def exported_symbols():
    import subprocess

    out = subprocess.check_output(["nm", "-D", "--defined-only", binding.lib_path()], text=True)
    return sorted({ln.split()[-1] for ln in out.splitlines() if ln.split()[-1].startswith("plssvm_")})


def test_library_loads_and_exports_every_declared_symbol():
    L = pl.load()
    decl = declared_symbols()
    assert len(decl) == 23
    for name in decl:
        assert hasattr(L, name), name
    assert exported_symbols() == decl  # nothing else is public
    assert sorted(binding.EXPORTS) == decl


def test_version_and_device_count():
    v = pl.plssvm_version()
    assert "sm_100a" in v and "NCCL 2." in v
    assert pl.plssvm_device_count() >= 0


def test_default_options():
    o = pl.options()
    assert (o.mode, o.x0, o.max_iter, o.replace_every, o.fixed_iter, o.device, o.device_pointers) == (0, 0, 0, 0, 0, 0, 0)
    assert o.stream is None and o.comm is None
    assert (o.cg_loop, o.multi_gpu) == (pl.CG_AUTO, pl.MULTI_GPU_ROWS)
    assert (o.num_gpus, o.transport, o.true_residual) == (0, pl.TRANSPORT_AUTO, 0)


def test_struct_layout_matches_header(tmp_path):
    """The binding's ctypes mirrors of plssvm_options_t / plssvm_stats_t have the header's size and
    field offsets (a C program compiled against include/plssvm.h prints them)."""
    import subprocess

    opts = [f for f, _ in binding.plssvm_options_t._fields_]
    stats = [f for f, _ in binding.plssvm_stats_t._fields_]
    src = tmp_path / "layout.c"
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "plssvm.h"', 'int main(void) {',
             'printf("%zu %zu\\n", sizeof(plssvm_options_t), sizeof(plssvm_stats_t));']
    lines += [f'printf("%zu\\n", offsetof(plssvm_options_t, {f}));' for f in opts]
    lines += [f'printf("%zu\\n", offsetof(plssvm_stats_t, {f}));' for f in stats]
    lines += ['return 0; }']
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    out = subprocess.check_output([str(exe)]).decode().split()
    so, ss = int(out[0]), int(out[1])
    assert so == ct.sizeof(binding.plssvm_options_t) and ss == ct.sizeof(binding.plssvm_stats_t)
    offs = [int(v) for v in out[2:]]
    assert offs[:len(opts)] == [getattr(binding.plssvm_options_t, f).offset for f in opts]
    assert offs[len(opts):] == [getattr(binding.plssvm_stats_t, f).offset for f in stats]


@pytest.mark.parametrize("m,P", [(2, 1), (256, 1), (16384, 1), (16384, 8), (1000, 3), (65536, 8), (131072, 8)])
def test_partition_rule(m, P):
    bands = [pl.plssvm_partition(m, P, r) for r in range(P)]
    mpad = bands[0][2]
    assert mpad % (128 * P) == 0 and mpad >= m and mpad - m < 128 * P
    assert bands[0][0] == 0 and bands[-1][1] == mpad
    for (b0, e0, _), (b1, e1, _) in zip(bands, bands[1:]):
        assert e0 == b1
    sizes = {e - b for b, e, _ in bands}
    assert len(sizes) == 1 and sizes.pop() % 128 == 0


@pytest.mark.parametrize("d,P", [(1, 1), (16, 1), (17, 2), (1024, 8), (4096, 8), (30, 4), (8, 8), (13, 3)])
def test_feature_partition_rule(d, P):
    """MULTI_GPU_FEATURES (paper §III-C5): contiguous feature slices covering [0, d)
    exactly once, sizes differing by at most one, none empty."""
    sl = [pl.plssvm_feature_partition(d, P, r) for r in range(P)]
    assert sl[0][0] == 0 and sl[-1][1] == d
    for (b0, e0), (b1, e1) in zip(sl, sl[1:]):
        assert e0 == b1
    sizes = [e - b for b, e in sl]
    assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1 and sum(sizes) == d


def test_feature_partition_invalid():
    with pytest.raises(pl.PlssvmError):
        pl.plssvm_feature_partition(3, 4, 0)  # d < P
    with pytest.raises(pl.PlssvmError):
        pl.plssvm_feature_partition(8, 2, 2)


def test_engine_options_validated():
    """Out-of-range engine / loop / variant options are rejected before any device work."""
    L = pl.load()
    X = np.random.default_rng(0).standard_normal((10, 3))
    y = np.array([1, -1] * 5, dtype=float)
    alpha, b = np.zeros(10), np.zeros(1)
    for kw in (dict(fp64_engine=3), dict(fp32_engine=4), dict(cg_loop=3), dict(cg_variant=2), dict(multi_gpu=2),
               dict(transport=3), dict(num_gpus=2, comm=1)):
        o = pl.options(**kw)
        st = L.plssvm_train_ex(X.ctypes.data, y.ctypes.data, 10, 3, 0, 2, 0.5, 3, 0.0, 1.0, 1e-10, ct.byref(o),
                               alpha.ctypes.data, b.ctypes.data, None)
        assert st == binding.E_INVALID_ARG, kw
        assert pl.plssvm_last_error()


def test_partition_invalid():
    with pytest.raises(pl.PlssvmError):
        pl.plssvm_partition(1, 1, 0)
    with pytest.raises(pl.PlssvmError):
        pl.plssvm_partition(100, 2, 2)


def _train_status(X, y, **kw):
    L = pl.load()
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    alpha = np.full(X.shape[0], 7.0)
    b = np.full(1, 7.0)
    args = dict(kernel=2, gamma=0.5, degree=3, coef0=0.0, C=1.0, eps=1e-10)
    args.update(kw)
    st = L.plssvm_train(X.ctypes.data, y.ctypes.data, X.shape[0], X.shape[1], args["kernel"], args["gamma"],
                        args["degree"], args["coef0"], args["C"], args["eps"], alpha.ctypes.data, b.ctypes.data)
    return st, pl.plssvm_last_error(), alpha, b


def test_validation_errors_leave_outputs_untouched():
    X = np.random.default_rng(0).standard_normal((10, 3))
    y = np.array([1, -1] * 5, dtype=float)
    cases = [
        (dict(C=0.0), binding.E_INVALID_ARG),
        (dict(C=-1.0), binding.E_INVALID_ARG),
        (dict(gamma=0.0), binding.E_INVALID_ARG),
        (dict(kernel=3), binding.E_INVALID_ARG),  # sigmoid is not a PLSSVM kernel
        (dict(kernel=1, degree=0), binding.E_INVALID_ARG),
        (dict(eps=0.0), binding.E_INVALID_ARG),
    ]
    for kw, code in cases:
        st, msg, alpha, b = _train_status(X, y, **kw)
        assert st == code and msg, (kw, st, msg)
        assert np.all(alpha == 7.0) and b[0] == 7.0
    st, msg, _, _ = _train_status(X[:1], y[:1])
    assert st == binding.E_INVALID_ARG


def _data_validation_cases():
    """Array contents (labels, finiteness) are validated on the device after staging
    (driver.cu validate_inputs): E_LABELS / E_INVALID_ARG with a GPU, E_CUDA without one."""
    X = np.random.default_rng(0).standard_normal((10, 3))
    y = np.array([1, -1] * 5, dtype=float)
    Xn = X.copy()
    Xn[3, 1] = np.nan
    return [((X, np.ones(10)), binding.E_LABELS, "both classes"),
            ((X, np.array([1, -1, 2, 1, 1, 1, -1, -1, 1, 1.0])), binding.E_LABELS, "+1 or -1"),
            ((Xn, y), binding.E_INVALID_ARG, "finite")]


@pytest.mark.skipif(pl.plssvm_device_count() > 0, reason="GPU present")
def test_data_validation_needs_the_device():
    for (X, y), _, _ in _data_validation_cases():
        st, msg, alpha, b = _train_status(X, y)
        assert st == binding.E_CUDA and np.all(alpha == 7.0) and b[0] == 7.0


@pytest.mark.gpu
def test_data_validation_on_device_leaves_outputs_untouched():
    for (X, y), code, text in _data_validation_cases():
        st, msg, alpha, b = _train_status(X, y)
        assert st == code and text in msg, (st, msg)
        assert np.all(alpha == 7.0) and b[0] == 7.0
    X = np.random.default_rng(1).standard_normal((10, 3))
    Z = X.copy()
    Z[2, 2] = np.inf
    with pytest.raises(pl.PlssvmError, match="Z is not finite"):
        pl.plssvm_predict(X, np.zeros(10), 0.0, Z, pl.RBF, 0.5)
    with pytest.raises(pl.PlssvmError, match="alpha is not finite"):
        pl.plssvm_predict(X, np.full(10, np.nan), 0.0, X, pl.RBF, 0.5)
    with pytest.raises(pl.PlssvmError, match="p is not finite"):
        pl.plssvm_qtilde_matvec(X, np.full(9, np.inf), pl.RBF, 0.5)
    import torch  # device pointers are validated too

    tX = torch.from_numpy(X).cuda()
    ty = torch.from_numpy(np.ones(10)).cuda()
    with pytest.raises(pl.PlssvmError, match="both classes"):
        pl.plssvm_train_ex(tX, ty, pl.RBF, 0.5)


def test_linear_kernel_ignores_gamma_validation():
    X = np.random.default_rng(0).standard_normal((10, 3))
    y = np.array([1, -1] * 5, dtype=float)
    st, msg, _, _ = _train_status(X, y, kernel=0, gamma=0.0)
    assert st in (binding.OK, binding.E_CUDA)


@pytest.mark.skipif(pl.plssvm_device_count() > 0, reason="GPU present")
def test_no_cpu_fallback_without_gpu():
    X = np.random.default_rng(0).standard_normal((10, 3))
    y = np.array([1, -1] * 5, dtype=float)
    st, msg, alpha, b = _train_status(X, y)
    assert st == binding.E_CUDA and "no CUDA device" in msg
    with pytest.raises(pl.PlssvmError):
        pl.plssvm_predict(X, np.zeros(10), 0.0, X, pl.RBF, 0.5)
    with pytest.raises(pl.PlssvmError):
        pl.plssvm_qtilde_matvec(X, np.zeros(9), pl.RBF, 0.5)

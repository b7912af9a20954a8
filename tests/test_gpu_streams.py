"""Stream ordering of device-pointer calls (plssvm.h options.stream; binding._device_opts).

torch's default stream has the handle 0, which the C ABI reads as "no stream" (the library's own
non-blocking stream, NOT ordered after other streams' work).  The binding therefore passes torch's
default stream as cudaStreamLegacy: a call that follows torch work on that stream without a
synchronisation must see its results.  The test makes the race real -- a spin kernel delays the
copy that writes X / p on torch's stream -- and checks the product against the oracle on the final
data (a call on an unordered stream would read the zeros)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2202_12674_b200 as pl

pytestmark = pytest.mark.gpu


def test_device_pointer_call_is_ordered_after_torch_default_stream():
    rng = np.random.default_rng(11)
    m, d = 1000, 64
    X = rng.standard_normal((m, d))
    p = rng.standard_normal(m - 1)
    src_X, src_p = torch.from_numpy(X).cuda(), torch.from_numpy(p).cuda()
    tX = torch.zeros_like(src_X)
    tp = torch.zeros_like(src_p)
    opts = lambda: pl.options(mode=pl.MODE_IMPLICIT, fp64_engine=pl.FP64_OZAKI)  # noqa: E731
    # warm-up call: the library's one-time setup (pinned staging buffers: cudaHostAlloc synchronises
    # the device) must not hide the race below
    pl.plssvm_qtilde_matvec(src_X, src_p, pl.RBF, 1.0 / d, 3, 0.0, 1.0, opts=opts())
    torch.cuda.synchronize()
    assert torch.cuda.current_stream().cuda_stream == 0  # the legacy default stream
    torch.cuda._sleep(200_000_000)  # ~0.1 s spin on torch's stream, then the real inputs land
    tX.copy_(src_X)
    tp.copy_(src_p)
    out, _ = pl.plssvm_qtilde_matvec(tX, tp, pl.RBF, 1.0 / d, 3, 0.0, 1.0, opts=opts())
    ref = oracle.qtilde(X, pl.RBF, 1.0 / d, 3, 0.0, 1.0) @ p
    got = out.cpu().numpy()
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref), np.linalg.norm(got - ref) / np.linalg.norm(ref)


def test_device_pointer_call_on_a_side_stream():
    """A torch side stream is passed through as is (work ordered on it; the call synchronises it)."""
    rng = np.random.default_rng(12)
    m, d = 700, 40
    X = rng.standard_normal((m, d))
    y = np.where(rng.random(m) < 0.5, 1.0, -1.0)
    y[0], y[1] = 1.0, -1.0
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        tX = torch.from_numpy(X).cuda()
        ty = torch.from_numpy(y).cuda()
        torch.cuda._sleep(100_000_000)
        tX2 = tX * 1.0  # written on s after the spin
        alpha, b, st, stats = pl.plssvm_train_ex(tX2, ty, pl.RBF, gamma=1.0 / d, eps=1e-10)
    a_ref, b_ref, _, _ = oracle.train(X, y, pl.RBF, 1.0 / d, 3, 0.0, 1.0, 1e-10)
    a = alpha.cpu().numpy()
    assert st == pl.OK
    assert np.linalg.norm(a - a_ref) <= 1e-7 * np.linalg.norm(a_ref)
    assert abs(float(b.item()) - b_ref) <= 1e-7 * max(abs(b_ref), np.abs(a_ref).max())

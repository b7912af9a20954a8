"""Chronopoulos-Gear single-reduction CG (options.cg_variant = SINGLE_REDUCTION, SURVEY §8(f)
NEXT-1) on the GPU: the same (alpha, b) as the oracle's Shewchuk CG (the unique Eq. 11
solution, <= 1e-7 at eps = 1e-10), iteration counts within a few of the Shewchuk loop, in every
product mode, with the batched and the CUDA-graph loop, and on several ranks (one all-reduce of
the (gamma, delta) pair per iteration)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2202_12674_b200 as pl
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _close(a, b, a_ref, b_ref, tol=1e-7):
    assert np.linalg.norm(a - a_ref) <= tol * np.linalg.norm(a_ref), np.linalg.norm(a - a_ref) / np.linalg.norm(a_ref)
    assert abs(b - b_ref) <= tol * max(abs(b_ref), np.abs(a_ref).max())


@pytest.mark.parametrize("kernel,mode,m,d,dtype", [
    (pl.LINEAR, pl.MODE_IMPLICIT, 256, 16, np.float64),      # C0 shape
    (pl.RBF, pl.MODE_IMPLICIT, 1000, 33, np.float64),
    (pl.RBF, pl.MODE_CACHED, 777, 20, np.float64),
    (pl.POLYNOMIAL, pl.MODE_CACHED, 900, 24, np.float64),
    (pl.LINEAR, pl.MODE_LOWRANK, 1200, 40, np.float64),
    (pl.POLYNOMIAL, pl.MODE_IMPLICIT, 640, 31, np.float32),
])
@pytest.mark.parametrize("loop", [pl.CG_BATCHED, pl.CG_GRAPH])
def test_single_reduction_cg_matches_oracle(kernel, mode, m, d, dtype, loop):
    X, y, _, _ = synth.planes(m, d, 16, seed=7 + kernel)
    X, y = X.astype(dtype), y.astype(dtype)
    eps = 1e-10 if dtype == np.float64 else 1e-6
    g = 1.0 / d
    a, b, st, s = pl.plssvm_train_ex(X, y, kernel, g, 3, 0.0, 1.0, eps,
                                     opts=pl.options(mode=mode, cg_loop=loop, cg_variant=pl.CG_SINGLE_REDUCTION))
    a2, b2, st2, s2 = pl.plssvm_train_ex(X, y, kernel, g, 3, 0.0, 1.0, eps, opts=pl.options(mode=mode, cg_loop=loop))
    assert st == st2 == 0
    assert abs(s.iterations - s2.iterations) <= max(2, 0.05 * s2.iterations)
    assert s.matvecs == s.iterations + 1 and s.rel_residual <= eps
    if dtype == np.float64:
        a_r, b_r, it_r, _ = oracle.train(X, y, kernel, g, 3, 0.0, 1.0, eps)
        _close(a, b, a_r, b_r)
    else:  # fp32: the product-level bar only; the two formulations agree to fp32 CG accuracy
        assert np.linalg.norm(a - a2) <= 1e-3 * np.linalg.norm(a2)


def test_single_reduction_cg_stops_and_options():
    X, y, _, _ = synth.planes(500, 12, 16, seed=3)
    a, b, st, s = pl.plssvm_train_ex(X, y, pl.RBF, 0.1, 3, 0.0, 1.0, 1e-14,
                                     opts=pl.options(mode=pl.MODE_IMPLICIT, max_iter=5, cg_variant=1))
    assert st == pl.binding.W_NOT_CONVERGED and s.iterations == 5
    a, b, st, s = pl.plssvm_train_ex(X, y, pl.RBF, 0.1, 3, 0.0, 1.0, 1e-10, opts=pl.options(fixed_iter=7, cg_variant=1))
    assert st == 0 and s.iterations == 7
    a, b, st, s = pl.plssvm_train_ex(X, y, pl.LINEAR, 1.0, 3, 0.0, 1.0, 1e-10, opts=pl.options(x0=1, cg_variant=1))
    a_r, b_r, _, _ = oracle.train(X, y, pl.LINEAR, 1.0, 3, 0.0, 1.0, 1e-10, x0=1)
    _close(a, b, a_r, b_r, tol=1e-6)  # x0 = ones: DESIGN.md R-5
    with pytest.raises(pl.PlssvmError):
        pl.plssvm_train_ex(X, y, pl.RBF, 0.1, 3, 0.0, 1.0, 1e-10, opts=pl.options(replace_every=5, cg_variant=1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, path, kernel, mode, m, d, mg):
    import sys

    sys.path.insert(0, ROOT)
    import paper_2202_12674_b200 as pl
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = pl.comm_host_staged(0, circulant=True)
    X, y, _, _ = synth.planes(m, d, 64, seed=40 + kernel)
    a, b, st, s = pl.plssvm_train_ex(X, y, kernel, 1.0 / d, 3, 0.5, 1.0, 1e-10,
                                     opts=pl.options(mode=mode, comm=comm, multi_gpu=mg, cg_variant=1))
    if rank == 0:
        np.savez(path, alpha=a, b=b, st=st, ranks=s.num_ranks)
    pl.plssvm_comm_destroy(comm)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kernel,mode,m,d,mg", [
    (2, pl.RBF, pl.MODE_IMPLICIT, 1000, 33, 0),   # circulant pairs + reduce-scatter
    (3, pl.RBF, pl.MODE_CACHED, 900, 20, 0),      # packed cached band
    (2, pl.LINEAR, pl.MODE_IMPLICIT, 800, 30, 1),  # the paper's feature split
])
def test_single_reduction_cg_multirank(tmp_path, world, kernel, mode, m, d, mg):
    path = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), path, kernel, mode, m, d, mg), nprocs=world, join=True)
    r = np.load(path)
    X, y, _, _ = synth.planes(m, d, 64, seed=40 + kernel)
    a_r, b_r, _, _ = oracle.train(X, y, kernel, 1.0 / d, 3, 0.5, 1.0, 1e-10)
    assert int(r["st"]) == 0 and int(r["ranks"]) == world
    _close(r["alpha"], float(r["b"]), a_r, b_r)


@pytest.mark.parametrize("mode,loop", [(pl.MODE_IMPLICIT, pl.CG_BATCHED), (pl.MODE_CACHED, pl.CG_AUTO)])
def test_residual_trace(mode, loop):
    """options.residual_trace (SURVEY §5 metrics, SPEC CGTrace): ||r_k|| for k = 0 .. iterations.  Pins:
    entry 0 is ||rhs|| (x0 = 0, Eq. 14); entry j equals the recurrence residual a run capped at j
    iterations stops with (the device path is deterministic, so bit for bit); the last entry is below the
    threshold eps ||r_0|| and the one before above it; and the same quantity recorded by the oracle's CG
    (sqrt(delta_k)) agrees over the first iterations (later the residual norm of CG is erratic on this
    system -- non-monotone peaks that two summation orders place an iteration apart -- while both runs
    stop within 2 iterations of each other)."""
    X, y, _, _ = synth.planes(700, 24, 16, seed=17)
    gamma, eps = 1.0 / 24, 1e-10

    def run(**kw):
        buf = np.full(400, -1.0)
        a, b, st, s = pl.plssvm_train_ex(X, y, pl.RBF, gamma, 3, 0.0, 1.0, eps,
                                         opts=pl.options(mode=mode, cg_loop=loop, residual_trace=buf.ctypes.data,
                                                         residual_trace_len=buf.size, **kw))
        return buf, st, s

    buf, st, s = run()
    assert st == 0 and s.cg_loop_used == pl.CG_BATCHED  # (a trace forces the batched loop)
    n = s.iterations + 1
    assert np.all(buf[:n] >= 0.0) and np.all(buf[n:] == -1.0)
    rhs = y[:-1] - y[-1]
    assert abs(buf[0] - np.linalg.norm(rhs)) <= 1e-13 * np.linalg.norm(rhs)
    assert buf[s.iterations] <= eps * buf[0] < buf[s.iterations - 1]
    for j in (1, 5, s.iterations // 2):
        bj, stj, sj = run(max_iter=j)
        assert sj.iterations == j and np.array_equal(bj[:j + 1], buf[:j + 1])
        assert sj.rel_residual * buf[0] == pytest.approx(buf[j], rel=1e-14)
    Qt = oracle.qtilde(X, pl.RBF, gamma, 3, 0.0, 1.0)
    _, it_ref, _, tr = oracle.cg(Qt, rhs, eps=eps, trace=True)
    assert abs(it_ref - s.iterations) <= 2
    np.testing.assert_allclose(buf[:5], tr[:5], rtol=1e-9)
    with pytest.raises(pl.PlssvmError, match="Shewchuk"):
        pl.plssvm_train_ex(X, y, pl.RBF, gamma, 3, 0.0, 1.0, eps,
                           opts=pl.options(cg_variant=pl.CG_SINGLE_REDUCTION, residual_trace=buf.ctypes.data,
                                           residual_trace_len=buf.size))

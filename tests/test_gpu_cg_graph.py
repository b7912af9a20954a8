"""CG loop as one CUDA graph (plssvm_cg_loop_t GRAPH): a device-side WHILE
conditional node repeats the iteration body until k_update_p's last block clears the condition
(Shewchuk's loop condition).  The graph issues exactly the kernels of the batched
host loop in the same order, so the trained model must be BIT-identical to BATCHED, and both
must match the oracle (alpha, b <= 1e-7 relative at eps = 1e-10, the north_star bar)."""

import numpy as np
import pytest

import oracle
import paper_2202_12674_b200 as pl
import synth

pytestmark = pytest.mark.gpu


def _train(X, y, kernel, gamma, eps, **kw):
    return pl.plssvm_train_ex(X, y, kernel, gamma, 3, 0.0, 1.0, eps, opts=pl.options(**kw))


@pytest.mark.parametrize("kernel,mode,m,d,dtype", [
    (pl.LINEAR, pl.MODE_IMPLICIT, 256, 16, np.float64),      # C0 shape
    (pl.RBF, pl.MODE_IMPLICIT, 1000, 33, np.float64),        # ragged, Ozaki engine
    (pl.RBF, pl.MODE_CACHED, 777, 20, np.float64),           # packed cached GEMV
    (pl.POLYNOMIAL, pl.MODE_CACHED, 900, 24, np.float64),
    (pl.LINEAR, pl.MODE_LOWRANK, 1200, 40, np.float64),      # O(md) product kernels
    (pl.POLYNOMIAL, pl.MODE_IMPLICIT, 640, 31, np.float32),  # tcgen05 3xTF32 engine
])
def test_graph_loop_bit_identical_to_batched_and_matches_oracle(kernel, mode, m, d, dtype):
    X, y, _, _ = synth.planes(m, d, 16, seed=7 + kernel)
    X, y = X.astype(dtype), y.astype(dtype)
    eps = 1e-10 if dtype == np.float64 else 1e-6
    g = 1.0 / d
    a_g, b_g, st_g, s_g = _train(X, y, kernel, g, eps, mode=mode, cg_loop=pl.CG_GRAPH)
    a_b, b_b, st_b, s_b = _train(X, y, kernel, g, eps, mode=mode, cg_loop=pl.CG_BATCHED)
    assert s_g.cg_loop_used == pl.CG_GRAPH and s_b.cg_loop_used == pl.CG_BATCHED
    assert st_g == st_b == 0 and s_g.iterations == s_b.iterations
    assert np.array_equal(a_g, a_b) and b_g == b_b
    # launches: the body's kernels once per iteration + the entry node
    assert s_g.gpu_launches >= s_g.iterations * 2  # product + the fused vector kernel (k_cg_fused)
    if dtype == np.float64:
        a_r, b_r, _, _ = oracle.train(X, y, kernel, g, 3, 0.0, 1.0, eps)
        assert np.linalg.norm(a_g - a_r) <= 1e-7 * np.linalg.norm(a_r)
        assert abs(b_g - b_r) <= 1e-7 * max(abs(b_r), np.abs(a_r).max())


def test_graph_loop_stops_at_max_iter_and_fixed_iter():
    X, y, _, _ = synth.planes(500, 12, 16, seed=3)
    a, b, st, s = _train(X, y, pl.RBF, 0.1, 1e-14, mode=pl.MODE_IMPLICIT, cg_loop=pl.CG_GRAPH, max_iter=5)
    assert st == pl.binding.W_NOT_CONVERGED and s.iterations == 5
    a2, b2, st2, s2 = _train(X, y, pl.RBF, 0.1, 1e-14, mode=pl.MODE_IMPLICIT, cg_loop=pl.CG_BATCHED, max_iter=5)
    assert st2 == st and np.array_equal(a, a2) and b == b2
    a3, b3, st3, s3 = _train(X, y, pl.RBF, 0.1, 1e-10, mode=pl.MODE_CACHED, cg_loop=pl.CG_GRAPH, fixed_iter=7)
    assert st3 == 0 and s3.iterations == 7


def test_graph_loop_x0_ones_and_auto_rule():
    X, y, _, _ = synth.planes(300, 10, 16, seed=11)
    a, b, st, s = _train(X, y, pl.LINEAR, 1.0, 1e-10, x0=1, cg_loop=pl.CG_GRAPH)
    a_r, b_r, _, _ = oracle.train(X, y, pl.LINEAR, 1.0, 3, 0.0, 1.0, 1e-10, x0=1)
    assert st == 0 and np.linalg.norm(a - a_r) <= 1e-7 * np.linalg.norm(a_r)
    # AUTO: small / cached problems run as a graph; residual replacement forces the batched loop
    _, _, _, s_auto = _train(X, y, pl.LINEAR, 1.0, 1e-10)
    assert s_auto.cg_loop_used == pl.CG_GRAPH
    _, _, _, s_rep = _train(X, y, pl.LINEAR, 1.0, 1e-10, replace_every=5)
    assert s_rep.cg_loop_used == pl.CG_BATCHED
    with pytest.raises(pl.PlssvmError):
        _train(X, y, pl.LINEAR, 1.0, 1e-10, replace_every=5, cg_loop=pl.CG_GRAPH)


def test_graph_loop_already_converged_start():
    """k_cg_start marks the loop done before the first iteration (imax = 1 with a huge eps
    after one step is the closest reachable case): the WHILE body must run 0 or 1 times and
    the graph must terminate."""
    X, y, _, _ = synth.planes(200, 5, 16, seed=2)
    a, b, st, s = _train(X, y, pl.RBF, 0.2, 0.9999, cg_loop=pl.CG_GRAPH)
    a2, b2, st2, s2 = _train(X, y, pl.RBF, 0.2, 0.9999, cg_loop=pl.CG_BATCHED)
    assert st == st2 and s.iterations == s2.iterations <= 2 and np.array_equal(a, a2)


@pytest.mark.parametrize("kernel,mode,m,d,dtype,loop", [
    (pl.RBF, pl.MODE_IMPLICIT, 1000, 33, np.float64, pl.CG_BATCHED),
    (pl.RBF, pl.MODE_IMPLICIT, 1000, 33, np.float64, pl.CG_GRAPH),
    (pl.POLYNOMIAL, pl.MODE_CACHED, 900, 24, np.float64, pl.CG_GRAPH),
    (pl.LINEAR, pl.MODE_LOWRANK, 1200, 40, np.float64, pl.CG_BATCHED),
    (pl.POLYNOMIAL, pl.MODE_IMPLICIT, 640, 31, np.float32, pl.CG_BATCHED),
    (pl.RBF, pl.MODE_CACHED, 777, 20, np.float32, pl.CG_GRAPH),
])
def test_fused_vector_kernel_bit_identical_to_three_kernels(kernel, mode, m, d, dtype, loop, monkeypatch):
    """k_cg_fused (finalize + update_xr + update_p in one cooperative launch, grid barriers in place of
    the kernel boundaries) performs the same arithmetic in the same order as the three kernels: the
    trained model is bit-identical; PLSSVM_CG_UNFUSED=1 selects the three-kernel sequence."""
    X, y, _, _ = synth.planes(m, d, 16, seed=5 + kernel)
    X, y = X.astype(dtype), y.astype(dtype)
    eps = 1e-10 if dtype == np.float64 else 1e-6
    a_f, b_f, st_f, s_f = _train(X, y, kernel, 1.0 / d, eps, mode=mode, cg_loop=loop)
    monkeypatch.setenv("PLSSVM_CG_UNFUSED", "1")
    a_u, b_u, st_u, s_u = _train(X, y, kernel, 1.0 / d, eps, mode=mode, cg_loop=loop)
    monkeypatch.delenv("PLSSVM_CG_UNFUSED")
    assert st_f == st_u == 0 and s_f.iterations == s_u.iterations
    assert np.array_equal(a_f, a_u) and b_f == b_u
    assert s_f.gpu_launches < s_u.gpu_launches

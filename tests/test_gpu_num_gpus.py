"""Single-process multi-GPU (options.num_gpus): one call drives P ranks, one host
thread each, with the library's PEER transport (peer copies + the all-gather of p fused into the CG
update kernel as direct stores into every rank's p).  On a one-GPU box the P ranks share cuda:0 --
the same driver code, the same collectives, the same fused stores (into buffers that happen to live
on one device); NCCL's ncclCommInitAll needs distinct devices and is checked for its refusal here.
Checks: trained (alpha, b) vs the oracle, the P-invariance of the model, predict labels, device
pointers, the stagnation guard, the true residual, and failure propagation between ranks."""
import numpy as np
import pytest

import oracle
import paper_2202_12674_b200 as pl
import synth

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def ndev():
    return pl.plssvm_device_count()


@pytest.mark.parametrize("P,kernel,mode,m,d", [
    (2, pl.RBF, pl.MODE_IMPLICIT, 1000, 33),      # circulant tile pairs + reduce-scatter, fused p
    (3, pl.POLYNOMIAL, pl.MODE_IMPLICIT, 900, 20),  # odd tile count, ragged
    (2, pl.LINEAR, pl.MODE_CACHED, 700, 17),      # packed circulant cached tiles
    (4, pl.RBF, pl.MODE_CACHED, 1500, 9),
    (3, pl.LINEAR, pl.MODE_LOWRANK, 1100, 30),    # all-reduce of X^T B p
])
def test_num_gpus_train_matches_oracle(P, kernel, mode, m, d):
    X, y, _, _ = synth.planes(m, d, 64, seed=41 + kernel)
    kw = dict(gamma=1.0 / d, degree=3, coef0=0.5)
    o = pl.options(mode=mode, num_gpus=P, transport=pl.TRANSPORT_PEER)
    alpha, b, st, s = pl.plssvm_train_ex(X, y, kernel, C=1.0, eps=1e-10, opts=o, **kw)
    a_ref, b_ref, _, _ = oracle.train(X, y, kernel, 1.0 / d, 3, 0.5, 1.0, 1e-10)
    assert st == 0 and s.num_ranks == P and s.mode_used == mode and s.transport_used == pl.TRANSPORT_PEER
    assert rel(alpha, a_ref) <= 1e-7
    assert abs(b - b_ref) <= 1e-7 * max(abs(b_ref), np.abs(a_ref).max())
    assert s.t_comm > 0.0
    # P-invariance (SURVEY §8(c) multi-GPU pin): only the summation order differs from one GPU
    a1, b1, st1, s1 = pl.plssvm_train_ex(X, y, kernel, C=1.0, eps=1e-10, opts=pl.options(mode=mode), **kw)
    assert abs(s1.iterations - s.iterations) <= 1
    assert rel(alpha, a1) <= 1e-9


@pytest.mark.parametrize("P", [2, 3])
def test_num_gpus_fp32_and_single_reduction(P):
    X, y, _, _ = synth.planes(1100, 37, 64, seed=5)
    X32, y32 = X.astype(np.float32), y.astype(np.float32)
    a1, b1, st1, _ = pl.plssvm_train_ex(X32, y32, pl.RBF, 1.0 / 37, eps=1e-6, opts=pl.options(mode=pl.MODE_IMPLICIT))
    a, b, st, s = pl.plssvm_train_ex(X32, y32, pl.RBF, 1.0 / 37, eps=1e-6,
                                     opts=pl.options(mode=pl.MODE_IMPLICIT, num_gpus=P))
    assert st == 0 and st1 == 0 and s.num_ranks == P
    assert rel(a, a1) <= 1e-3  # fp32 CG accuracy (R-12)
    # Chronopoulos-Gear on P ranks (copy-based all-gather, one all-reduce of the scalar pair)
    a_ref, b_ref, _, _ = oracle.train(X, y, pl.RBF, 1.0 / 37, eps=1e-10)
    a2, b2, st2, s2 = pl.plssvm_train_ex(X, y, pl.RBF, 1.0 / 37, eps=1e-10,
                                         opts=pl.options(num_gpus=P, cg_variant=pl.CG_SINGLE_REDUCTION, mode=1))
    assert st2 == 0 and rel(a2, a_ref) <= 1e-7


def test_num_gpus_device_pointers_and_predict():
    import torch

    X, y, Z, _ = synth.planes(1200, 24, 333, seed=8)
    tX, ty, tZ = (torch.from_numpy(a).cuda() for a in (X, y, Z))
    o = pl.options(mode=pl.MODE_IMPLICIT, num_gpus=2)
    alpha, b, st, s = pl.plssvm_train_ex(tX, ty, pl.RBF, 1.0 / 24, eps=1e-10, opts=o)
    a_ref, b_ref, _, _ = oracle.train(X, y, pl.RBF, 1.0 / 24, eps=1e-10)
    assert st == 0 and rel(alpha.cpu().numpy(), a_ref) <= 1e-7
    f_ref, lab_ref = oracle.predict(X, a_ref, b_ref, Z, pl.RBF, 1.0 / 24)
    for P in (2, 3):  # 333 test points split 111 / 111 / 111 and 166 / 167
        f, lab, _ = pl.plssvm_predict_ex(tX, alpha, float(b.item()), tZ, pl.RBF, 1.0 / 24,
                                         opts=pl.options(num_gpus=P))
        assert np.array_equal(lab.cpu().numpy(), lab_ref)
        assert np.max(np.abs(f.cpu().numpy() - f_ref)) <= 1e-9 * max(1.0, np.abs(f_ref).max())
    # host buffers, more ranks than test points
    f, lab = pl.plssvm_predict(X, a_ref, b_ref, Z[:2], pl.RBF, 1.0 / 24)
    f3, lab3, _ = pl.plssvm_predict_ex(X, a_ref, b_ref, Z[:2], pl.RBF, 1.0 / 24, opts=pl.options(num_gpus=3))
    assert np.array_equal(lab, lab3) and np.max(np.abs(f - f3)) <= 1e-12 * max(1.0, np.abs(f).max())


def test_num_gpus_nccl_needs_distinct_devices():
    if ndev() >= 2:
        pytest.skip("more than one device: NCCL is allowed")
    X, y, _, _ = synth.planes(300, 8, 0, seed=1)
    with pytest.raises(pl.PlssvmError) as e:
        pl.plssvm_train_ex(X, y, pl.RBF, 0.125, opts=pl.options(num_gpus=2, transport=pl.TRANSPORT_NCCL))
    assert e.value.status == pl.E_INVALID_ARG
    # AUTO picks the peer transport when ranks share a device
    a, b, st, s = pl.plssvm_train_ex(X, y, pl.RBF, 0.125, opts=pl.options(num_gpus=2))
    assert st == 0 and s.transport_used == pl.TRANSPORT_PEER
    # one rank through ncclCommInitAll (the only NCCL configuration a one-GPU box can run)
    a1, b1, st1, s1 = pl.plssvm_train_ex(X, y, pl.RBF, 0.125, opts=pl.options(num_gpus=1, transport=pl.TRANSPORT_NCCL))
    assert st1 == 0 and rel(a1, a) <= 1e-9


def test_num_gpus_failure_is_reported_once():
    X, y, _, _ = synth.planes(400, 8, 0, seed=2)
    y = y.copy()
    y[17] = 0.5  # invalid label: every rank's validation fails; the call reports one error
    with pytest.raises(pl.PlssvmError) as e:
        pl.plssvm_train_ex(X, y, pl.RBF, 0.125, opts=pl.options(num_gpus=3))
    assert e.value.status == pl.E_LABELS and "rank" in str(e.value)
    with pytest.raises(pl.PlssvmError) as e:
        pl.plssvm_train_ex(X, y, pl.RBF, 0.125, opts=pl.options(num_gpus=2, comm=1))
    assert e.value.status == pl.E_INVALID_ARG


def test_env_num_gpus(monkeypatch):
    X, y, _, _ = synth.planes(500, 12, 0, seed=3)
    monkeypatch.setenv("PLSSVM_NUM_GPUS", "2")
    a, b, st, s = pl.plssvm_train_ex(X, y, pl.RBF, 1.0 / 12, eps=1e-10, opts=pl.options(mode=pl.MODE_IMPLICIT))
    assert st == 0 and s.num_ranks == 2
    a2, b2, st2 = pl.plssvm_train(X, y, pl.RBF, 1.0 / 12, eps=1e-10)  # plain entry point: env too
    monkeypatch.delenv("PLSSVM_NUM_GPUS")
    a1, b1, st1, s1 = pl.plssvm_train_ex(X, y, pl.RBF, 1.0 / 12, eps=1e-10, opts=pl.options(mode=pl.MODE_IMPLICIT))
    assert s1.num_ranks == 1 and rel(a, a1) <= 1e-9 and rel(a2, a1) <= 1e-7


# ---------------------------------------------------------------- a5: stagnation guard, true residual
@pytest.mark.parametrize("P", [1, 2])
def test_stagnation_guard_device(P):
    """DESIGN.md R-20: with residual replacement on and an unreachable eps the device loop
    stops with W_NOT_CONVERGED / STOP_STAGNATED long before imax, like the oracle; the model is still the
    KKT solution to ~kappa u."""
    X, y, _, _ = synth.planes(600, 16, 0, seed=12)
    kw = dict(gamma=1.0 / 16)
    a_ref, b_ref, it_ref, st_ref = oracle.train(X, y, pl.RBF, C=1.0, eps=1e-17, replace_every=5, **kw)
    assert st_ref == oracle.W_NOT_CONVERGED and it_ref < 599
    a, b, st, s = pl.plssvm_train_ex(X, y, pl.RBF, C=1.0, eps=1e-17, **kw,
                                     opts=pl.options(mode=pl.MODE_IMPLICIT, replace_every=5, num_gpus=P))
    assert st == pl.W_NOT_CONVERGED and s.stop_reason == pl.STOP_STAGNATED
    assert s.iterations < 599 and abs(s.iterations - it_ref) <= max(10, it_ref // 4)
    assert rel(a, a_ref) <= 1e-8  # both at the attainable accuracy (~kappa u), far inside the 1e-7 bar
    # converging runs never see the guard
    a, b, st, s = pl.plssvm_train_ex(X, y, pl.RBF, C=1.0, eps=1e-10, **kw, opts=pl.options(replace_every=5))
    assert st == 0 and s.stop_reason == pl.STOP_CONVERGED


@pytest.mark.parametrize("mode", [pl.MODE_IMPLICIT, pl.MODE_CACHED])
def test_true_residual(mode):
    X, y, _, _ = synth.planes(900, 20, 0, seed=13)
    a, b, st, s = pl.plssvm_train_ex(X, y, pl.RBF, 0.05, eps=1e-10, opts=pl.options(mode=mode, true_residual=1))
    Qt = oracle.qtilde(X, pl.RBF, 0.05)
    rhs = y[:-1] - y[-1]
    true = np.linalg.norm(rhs - Qt @ a[:-1]) / np.linalg.norm(rhs)
    assert st == 0 and s.rel_residual <= 1e-10
    assert abs(s.rel_residual_true - true) <= 1e-3 * true + 1e-14
    assert s.matvecs == s.iterations + 1
    a2, b2, st2, s2 = pl.plssvm_train_ex(X, y, pl.RBF, 0.05, eps=1e-10, opts=pl.options(mode=mode))
    assert s2.rel_residual_true == -1.0 and np.array_equal(a, a2)


def test_breakdown_names_the_iteration():
    """p.Q~p <= 0 -> PLSSVM_E_NUMERICAL with a message naming the iteration.
    A polynomial kernel with coef0 < 0 and an even degree makes Q~ indefinite (R-17)."""
    rng = np.random.default_rng(4)
    X = rng.standard_normal((300, 6))
    y = np.where(rng.random(300) < 0.5, 1.0, -1.0)
    y[0], y[1] = 1.0, -1.0
    _, _, _, st_ref = oracle.train(X, y, pl.POLYNOMIAL, 1.0, 2, -6.0, 100.0, 1e-10)
    assert st_ref == oracle.E_NUMERICAL
    with pytest.raises(pl.PlssvmError) as e:
        pl.plssvm_train_ex(X, y, pl.POLYNOMIAL, 1.0, 2, -6.0, 100.0, 1e-10, opts=pl.options(mode=pl.MODE_IMPLICIT))
    assert e.value.status == pl.E_NUMERICAL and "iteration" in str(e.value)

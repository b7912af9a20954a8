"""Row-sharded multi-rank driver on real kernels: P processes share cuda:0 and exchange through
a host-staged torch.distributed (gloo) communicator (`comm_host_staged`; NCCL refuses two
ranks on one device).  The driver code path is the multi-GPU one (bands, out-of-band
row-only tiles, in-place all-gather of p, scalar all-reduces); only the transport differs
from NCCL.  Checks: the gathered product and the trained (alpha, b) against the oracle."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, path, kernel, mode, m, d, circ, mg=0, x0=0, f32=0):
    import sys

    sys.path.insert(0, ROOT)
    import paper_2202_12674_b200 as pl
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = pl.comm_host_staged(0, circulant=circ)
    X, y, Z, _ = synth.planes(m, d, 64, seed=21 + kernel)
    p = np.random.default_rng(5).standard_normal(m - 1)
    if f32:
        X, y, p = X.astype(np.float32), y.astype(np.float32), p.astype(np.float32)
    opts = pl.options(mode=mode, comm=comm, multi_gpu=mg)
    out, _ = pl.plssvm_qtilde_matvec(X, p, kernel, 1.0 / d, 3, 0.5, 1.0, opts=opts)
    alpha, b, st, stats = pl.plssvm_train_ex(X, y, kernel, 1.0 / d, 3, 0.5, 1.0, 1e-6 if f32 else 1e-10,
                                             opts=pl.options(mode=mode, comm=comm, multi_gpu=mg, x0=x0))
    if rank == 0:
        np.savez(path, out=out, alpha=alpha, b=b, st=st, it=stats.iterations, ranks=stats.num_ranks,
                 mode_used=stats.mode_used, tcomm=stats.t_comm, tcg=stats.t_cg)
    pl.plssvm_comm_destroy(comm)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("circ", [True, False])
@pytest.mark.parametrize("world,kernel,mode,m,d", [
    (2, 2, 1, 1000, 33),    # RBF implicit, m_pad = 1024 -> 4 tiles per band
    (2, 0, 2, 700, 17),     # linear cached
    (3, 1, 1, 900, 20),     # poly implicit, 3 ranks, ragged tail, odd T (9 tiles)
    (4, 2, 2, 1500, 9),     # RBF cached, 4 ranks
    (4, 2, 1, 2000, 40),    # RBF implicit, 4 ranks, T = 16 (circulant j = T/2 pairs)
    (3, 0, 3, 1100, 30),    # linear LOWRANK, 3 ranks (all-reduce of X^T B p)
])
def test_row_sharded_train_matches_oracle(tmp_path, world, kernel, mode, m, d, circ):
    """circ=True: implicit products use circulant tile pairs + reduce-scatter (cached: packed
    circulant tiles); False: row bands (cached: full rows per rank)."""
    if mode == 3 and not circ:
        pytest.skip("the low-rank mode does not use the reduce-scatter")
    # cached + circ: symmetric-packed tiles (circulant pairs) + reduce-scatter;
    # cached without a reduce-scatter: full-row bands
    import oracle
    import synth

    path = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), path, kernel, mode, m, d, circ), nprocs=world, join=True)
    r = np.load(path)
    X, y, _, _ = synth.planes(m, d, 64, seed=21 + kernel)
    p = np.random.default_rng(5).standard_normal(m - 1)
    Qt = oracle.qtilde(X, kernel, 1.0 / d, 3, 0.5, 1.0)
    ref = Qt @ p
    assert np.linalg.norm(r["out"] - ref) <= 1e-12 * np.linalg.norm(ref)
    a_ref, b_ref, it_ref, _ = oracle.train(X, y, kernel, 1.0 / d, 3, 0.5, 1.0, 1e-10)
    assert int(r["st"]) == 0 and int(r["ranks"]) == world and int(r["mode_used"]) == mode
    assert np.linalg.norm(r["alpha"] - a_ref) <= 1e-7 * np.linalg.norm(a_ref)
    assert abs(float(r["b"]) - b_ref) <= 1e-7 * max(abs(b_ref), np.abs(a_ref).max())
    # the collectives are timed separately: positive, inside the CG time
    assert 0.0 < float(r["tcomm"]) < float(r["tcg"])


@pytest.mark.parametrize("world,m,d,x0", [
    (2, 1000, 33, 0),   # ragged features (17 + 16), ragged points
    (3, 700, 20, 0),    # 3 ranks: 6 + 7 + 7 features
    (4, 1500, 9, 0),    # 4 ranks, 2-3 features each (smaller than one 32-feature slab)
    (2, 900, 64, 1),    # x0 = ones: initial product through the all-reduce too
])
def test_feature_split_train_matches_oracle(tmp_path, world, m, d, x0):
    """MULTI_GPU_FEATURES (paper §III-C5): every rank computes the partial Q~p of its
    feature slice (1/C terms on rank 0 only), one all-reduce per product; linear kernel."""
    import oracle
    import synth

    path = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), path, 0, 0, m, d, True, 1, x0), nprocs=world, join=True)
    r = np.load(path)
    X, y, _, _ = synth.planes(m, d, 64, seed=21)
    p = np.random.default_rng(5).standard_normal(m - 1)
    ref = oracle.qtilde(X, 0, 1.0 / d, 3, 0.5, 1.0) @ p
    assert np.linalg.norm(r["out"] - ref) <= 1e-12 * np.linalg.norm(ref)
    a_ref, b_ref, _, _ = oracle.train(X, y, 0, 1.0 / d, 3, 0.5, 1.0, 1e-10, x0=x0)
    assert int(r["st"]) == 0 and int(r["ranks"]) == world and int(r["mode_used"]) == 1
    # x0 = ones stops at eps relative to ||rhs - Q~1|| >> ||rhs||, so two summation orders agree
    # only to ~1e-6 on this linear system (R-5); x0 = 0: the 1e-7 bar
    tol = 1e-7 if x0 == 0 else 1e-6
    assert np.linalg.norm(r["alpha"] - a_ref) <= tol * np.linalg.norm(a_ref)
    assert abs(float(r["b"]) - b_ref) <= tol * max(abs(b_ref), np.abs(a_ref).max())


@pytest.mark.parametrize("world,kernel,mode", [(2, 1, 1), (3, 2, 1), (2, 2, 2)])
def test_fp32_int8_engine_multirank(tmp_path, world, kernel, mode):
    """fp32 (default AUTO -> the int8 3-digit engine) on several ranks: the gathered product vs the
    oracle (<= 1e-5) and the model vs the same engine on one rank (fp32 CG accuracy)."""
    import oracle
    import paper_2202_12674_b200 as pl
    import synth

    m, d = 1100, 37
    path = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), path, kernel, mode, m, d, True, 0, 0, 1), nprocs=world, join=True)
    r = np.load(path)
    X, y, _, _ = synth.planes(m, d, 64, seed=21 + kernel)
    X, y = X.astype(np.float32), y.astype(np.float32)
    p = np.random.default_rng(5).standard_normal(m - 1).astype(np.float32)
    gamma = float(np.float32(1.0 / d))
    ref = oracle.qtilde(X.astype(np.float64), kernel, gamma, 3, 0.5, 1.0) @ p.astype(np.float64)
    assert np.linalg.norm(r["out"] - ref) <= 1e-5 * np.linalg.norm(ref)
    a1, b1, st1, _ = pl.plssvm_train_ex(X, y, kernel, 1.0 / d, 3, 0.5, 1.0, 1e-6, opts=pl.options(mode=mode))
    assert int(r["st"]) == 0 and st1 == 0 and int(r["ranks"]) == world
    assert np.linalg.norm(r["alpha"] - a1) <= 1e-3 * np.linalg.norm(a1)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_p_invariance_of_the_trained_model(tmp_path, world):
    """SURVEY §8(c) multi-GPU pin: the row sharding changes only the summation order (DESIGN.md
    R-16), so the model trained on P ranks equals the one-GPU model far inside the parity bar
    (RBF, well conditioned: <= 1e-10 relative), with the same iteration count up to 1."""
    import paper_2202_12674_b200 as pl
    import synth

    m, d = 1000, 33
    path = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), path, 2, 1, m, d, True), nprocs=world, join=True)
    r = np.load(path)
    X, y, _, _ = synth.planes(m, d, 64, seed=21 + 2)
    a1, b1, st1, s1 = pl.plssvm_train_ex(X, y, 2, 1.0 / d, 3, 0.5, 1.0, 1e-10, opts=pl.options(mode=1))
    assert int(r["st"]) == 0 and st1 == 0 and abs(int(r["it"]) - s1.iterations) <= 1
    assert np.linalg.norm(r["alpha"] - a1) <= 1e-10 * np.linalg.norm(a1)
    assert abs(float(r["b"]) - b1) <= 1e-10 * max(abs(b1), np.abs(a1).max())


def _worker_nccl1(rank, world, port, path):
    import sys

    sys.path.insert(0, ROOT)
    import torch

    import paper_2202_12674_b200 as pl
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    comm = pl.comm_from_torch_distributed(0)  # NCCL unique id broadcast through torch.distributed
    X, y, _, _ = synth.planes(900, 20, 64, seed=31)
    p = np.random.default_rng(3).standard_normal(899)
    out, _ = pl.plssvm_qtilde_matvec(X, p, pl.RBF, 0.05, opts=pl.options(mode=pl.MODE_IMPLICIT, comm=comm))
    res = {}
    for name, kw in (("implicit", dict(mode=pl.MODE_IMPLICIT)), ("cached", dict(mode=pl.MODE_CACHED)),
                     ("cgcg", dict(mode=pl.MODE_IMPLICIT, cg_variant=pl.CG_SINGLE_REDUCTION)),
                     ("nolsa", dict(mode=pl.MODE_IMPLICIT))):
        if name == "nolsa":  # the separate ncclAllGather of p instead of the device-API stores
            os.environ["PLSSVM_NO_LSA"] = "1"
        a, b, st, s = pl.plssvm_train_ex(X, y, pl.RBF, 0.05, eps=1e-10, opts=pl.options(comm=comm, **kw))
        os.environ.pop("PLSSVM_NO_LSA", None)
        res[name] = (a, b, st, s.num_ranks, s.allgather_fused)
    np.savez(path, out=out, **{f"{k}_a": v[0] for k, v in res.items()}, **{f"{k}_b": v[1] for k, v in res.items()},
             **{f"{k}_st": v[2] for k, v in res.items()}, **{f"{k}_r": v[3] for k, v in res.items()},
             **{f"{k}_fused": v[4] for k, v in res.items()})
    pl.plssvm_comm_destroy(comm)
    dist.destroy_process_group()


def test_nccl_communicator_one_rank(tmp_path):
    """The NCCL transport itself (plssvm_comm_init through torch.distributed's id broadcast,
    ncclAllGather in place, ncclAllReduce out of place, the device-API fused all-gather of p) on a 1-rank communicator -- the one NCCL
    configuration a single-GPU box can run (NCCL refuses two ranks on one device); the multi-rank
    driver logic is covered above through the host-staged transport."""
    import oracle
    import synth

    path = str(tmp_path / "r.npz")
    mp.spawn(_worker_nccl1, args=(1, _free_port(), path), nprocs=1, join=True)
    r = np.load(path)
    X, y, _, _ = synth.planes(900, 20, 64, seed=31)
    p = np.random.default_rng(3).standard_normal(899)
    ref = oracle.qtilde(X, 2, 0.05) @ p
    assert np.linalg.norm(r["out"] - ref) <= 1e-12 * np.linalg.norm(ref)
    a_ref, b_ref, _, _ = oracle.train(X, y, 2, 0.05, eps=1e-10)
    for k in ("implicit", "cached", "cgcg", "nolsa"):
        assert int(r[f"{k}_st"]) == 0 and int(r[f"{k}_r"]) == 1
        assert np.linalg.norm(r[f"{k}_a"] - a_ref) <= 1e-7 * np.linalg.norm(a_ref), k
        assert abs(float(r[f"{k}_b"]) - b_ref) <= 1e-7 * max(abs(b_ref), np.abs(a_ref).max()), k
    # NCCL device API: p in the communicator's symmetric window, the all-gather
    # fused into the p update (LSA stores + barrier) for the Shewchuk loop; the same iterates as the
    # separate ncclAllGather, bit for bit
    assert int(r["implicit_fused"]) == 1 and int(r["cached_fused"]) == 1
    assert int(r["cgcg_fused"]) == 0 and int(r["nolsa_fused"]) == 0
    assert np.array_equal(r["implicit_a"], r["nolsa_a"]) and float(r["implicit_b"]) == float(r["nolsa_b"])

"""World-size-2 (gloo, CPU) check of the row-sharded multi-GPU host logic.

Each rank takes its band from the library's host rule `plssvm_partition`, computes its rows
of Q~p from the oracle's rows (a stand-in for the device product), and runs the same
per-iteration exchange sequence as the driver: all-gather of p, all-reduce of p.Ap and of
delta.  The assembled solution must equal the single-process oracle CG, and the gathered
product the full product."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    import sys

    sys.path.insert(0, ROOT)
    import oracle
    import paper_2202_12674_b200 as pl
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, y, _, _ = synth.planes(300, 7, seed=3)
    m = X.shape[0]
    m1 = m - 1
    b0, b1, mpad = pl.plssvm_partition(m, world, rank)
    nb = b1 - b0
    rows = np.arange(b0, b1)
    valid = rows < m1
    R = np.zeros((nb, m1))
    R[valid] = oracle.qtilde_rows(X, rows[valid], oracle.RBF, 0.2, C=1.0)

    def band_product(pfull):  # this rank's rows of Q~ p (padding rows are 0)
        return R @ pfull[:m1]

    def allgather(band):
        out = [torch.zeros(nb, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(band.copy()))
        return torch.cat(out).numpy()

    def allreduce(v):
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())

    # product check
    p = np.random.default_rng(1).standard_normal(mpad)
    p[m1:] = 0.0
    yfull = allgather(band_product(p))
    # sharded CG (driver sequence), x0 = 0
    rhs = np.where(valid, y[np.minimum(rows, m - 1)] - y[m - 1], 0.0)
    x = np.zeros(nb)
    r = rhs.copy()
    pb = r.copy()
    delta = allreduce(r @ r)
    delta0 = delta
    it = 0
    while it < m1 and delta > 1e-20 * delta0:
        pf = allgather(pb)
        yb = band_product(pf)
        pap = allreduce(pb @ yb)
        a = delta / pap
        x += a * pb
        r -= a * yb
        dnew = allreduce(r @ r)
        pb = r + (dnew / delta) * pb
        delta = dnew
        it += 1
    xfull = allgather(x)[:m1]
    if rank == 0:
        Qt = oracle.qtilde(X, oracle.RBF, 0.2, C=1.0)
        ref_y = Qt @ p[:m1]
        xo, ito, st = oracle.cg(Qt, y[:-1] - y[-1], eps=1e-10)
        np.savez(result_path, y=yfull[:m1], ref_y=ref_y, x=xfull, ref_x=xo, it=it, ito=ito, mpad=mpad)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_sharded_cg_gloo(tmp_path, world):
    path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    res = np.load(path)
    assert res["mpad"] % (128 * world) == 0
    assert np.linalg.norm(res["y"] - res["ref_y"]) <= 1e-13 * np.linalg.norm(res["ref_y"])
    assert np.linalg.norm(res["x"] - res["ref_x"]) <= 1e-8 * np.linalg.norm(res["ref_x"])
    assert abs(int(res["it"]) - int(res["ito"])) <= 2


def circulant_pairs(T, P):
    """The circulant rule of driver.cu circulant_tiles(): tile row I owns (I, (I+j) % T),
    j = 0..T/2, the pair j = T/2 (even T) only for I < T/2; rank r takes rows [r T/P, (r+1) T/P)."""
    per = T // P
    out = []
    for r in range(P):
        tiles = []
        for I in range(r * per, (r + 1) * per):
            for j in range(T // 2 + 1):
                if T % 2 == 0 and j == T // 2 and I >= T // 2:
                    continue
                J = (I + j) % T
                if j > 0 and J == I:
                    continue
                tiles.append((I, J))
        out.append(tiles)
    return out


@pytest.mark.parametrize("T,P", [(8, 2), (9, 3), (16, 4), (64, 8), (1024, 8), (128, 1)])
def test_circulant_pairs_cover_each_unordered_pair_once_and_balance(T, P):
    ranks = circulant_pairs(T, P)
    seen = {}
    for tiles in ranks:
        for I, J in tiles:
            key = (min(I, J), max(I, J))
            seen[key] = seen.get(key, 0) + 1
    assert len(seen) == T * (T + 1) // 2 and set(seen.values()) == {1}
    loads = [len(t) for t in ranks]
    assert max(loads) / min(loads) <= 1 + 2.0 / T + 1e-12 or T < 16


def _worker_features(rank, world, port, result_path):
    """MULTI_GPU_FEATURES host logic (paper §III-C5): rank g holds the feature slice
    from plssvm_feature_partition and forms its partial Q~^(g) of Eq. 16 on that slice, with
    the 1/C terms on rank 0 only (C = inf elsewhere); one all-reduce of the partial products per
    iteration, replicated CG vectors.  Must reproduce the single-process Q~p and CG solution."""
    import sys

    sys.path.insert(0, ROOT)
    import oracle
    import paper_2202_12674_b200 as pl
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, y, _, _ = synth.planes(260, 11, seed=4)
    m1 = X.shape[0] - 1
    f0, f1 = pl.plssvm_feature_partition(X.shape[1], world, rank)
    Qg = oracle.qtilde(np.ascontiguousarray(X[:, f0:f1]), oracle.LINEAR, C=2.0 if rank == 0 else np.inf)

    def product(p):  # partial product of this slice, summed over the ranks
        t = torch.from_numpy(Qg @ p)
        dist.all_reduce(t)
        return t.numpy()

    p = np.random.default_rng(2).standard_normal(m1)
    yfull = product(p)
    rhs = y[:-1] - y[-1]
    x = np.zeros(m1)
    r = rhs.copy()
    pv = r.copy()
    delta = delta0 = r @ r
    it = 0
    while it < m1 and delta > 1e-20 * delta0:
        yv = product(pv)
        a = delta / (pv @ yv)
        x += a * pv
        r -= a * yv
        dnew = r @ r
        pv = r + (dnew / delta) * pv
        delta = dnew
        it += 1
    if rank == 0:
        Qt = oracle.qtilde(X, oracle.LINEAR, C=2.0)
        xo, ito, _ = oracle.cg(Qt, rhs, eps=1e-10)
        np.savez(result_path, y=yfull, ref_y=Qt @ p, x=x, ref_x=xo, it=it, ito=ito)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_feature_split_cg_gloo(tmp_path, world):
    path = str(tmp_path / "res.npz")
    mp.spawn(_worker_features, args=(world, _free_port(), path), nprocs=world, join=True)
    res = np.load(path)
    assert np.linalg.norm(res["y"] - res["ref_y"]) <= 1e-13 * np.linalg.norm(res["ref_y"])
    assert np.linalg.norm(res["x"] - res["ref_x"]) <= 1e-8 * np.linalg.norm(res["ref_x"])
    assert abs(int(res["it"]) - int(res["ito"])) <= 2


def _worker_cgcg(rank, world, port, result_path):
    """Chronopoulos-Gear CG with the driver's exchange sequence (kernels.cuh k_cgcg_update): per
    iteration ONE all-gather of r, the band product w = (Q~ r)_band, and ONE all-reduce of the
    pair (gamma, delta).  Must reach the single-process oracle CG solution."""
    import sys

    sys.path.insert(0, ROOT)
    import oracle
    import paper_2202_12674_b200 as pl
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, y, _, _ = synth.planes(300, 7, seed=3)
    m = X.shape[0]
    m1 = m - 1
    b0, b1, mpad = pl.plssvm_partition(m, world, rank)
    nb = b1 - b0
    rows = np.arange(b0, b1)
    valid = rows < m1
    R = np.zeros((nb, m1))
    R[valid] = oracle.qtilde_rows(X, rows[valid], oracle.RBF, 0.2, C=1.0)

    def allgather(band):
        out = [torch.zeros(nb, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(band.copy()))
        return torch.cat(out).numpy()

    def allreduce_pair(a, b):
        t = torch.tensor([a, b], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t[0]), float(t[1])

    reductions = 0
    r = np.where(valid, y[np.minimum(rows, m - 1)] - y[m - 1], 0.0)
    x = np.zeros(nb)
    p = np.zeros(nb)
    s = np.zeros(nb)
    gamma, _ = allreduce_pair(r @ r, 0.0)
    thr = 1e-20 * gamma
    it, g_prev, a_prev = 0, 0.0, 0.0
    while True:
        w = R @ allgather(r)[:m1]
        gamma, delta = allreduce_pair(r @ r, w @ r)  # the one reduction point
        reductions += 1
        if gamma <= thr or it >= m1:
            break
        beta = gamma / g_prev if it > 0 else 0.0
        alpha = gamma / (delta - beta * gamma / a_prev) if it > 0 else gamma / delta
        p = r + beta * p
        s = w + beta * s
        x += alpha * p
        r = r - alpha * s
        g_prev, a_prev = gamma, alpha
        it += 1
    xfull = allgather(x)[:m1]
    if rank == 0:
        Qt = oracle.qtilde(X, oracle.RBF, 0.2, C=1.0)
        xo, ito, _ = oracle.cg(Qt, y[:-1] - y[-1], eps=1e-10)
        np.savez(result_path, x=xfull, ref_x=xo, it=it, ito=ito, red=reductions)
    dist.barrier()
    dist.destroy_process_group()


def test_single_reduction_cg_gloo(tmp_path):
    path = str(tmp_path / "res.npz")
    mp.spawn(_worker_cgcg, args=(2, _free_port(), path), nprocs=2, join=True)
    res = np.load(path)
    assert np.linalg.norm(res["x"] - res["ref_x"]) <= 1e-8 * np.linalg.norm(res["ref_x"])
    assert abs(int(res["it"]) - int(res["ito"])) <= 2
    assert int(res["red"]) == int(res["it"]) + 1  # one all-reduce per iteration (+ the final test)

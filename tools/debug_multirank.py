"""Debug helper: 2 ranks on one GPU (host-staged gloo comm), print the training stats."""
import os
import socket
import sys

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, world, port, mode, kernel, m, d):
    sys.path.insert(0, ROOT)
    import paper_2202_12674_b200 as pl
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = pl.comm_host_staged(0)
    X, y, Z, _ = synth.planes(m, d, 64, seed=21 + kernel)
    a, b, st, s = pl.plssvm_train_ex(X, y, kernel, 1.0 / d, 3, 0.5, 1.0, 1e-10, opts=pl.options(mode=mode, comm=comm))
    a2, b2, st2, s2 = pl.plssvm_train_ex(X, y, kernel, 1.0 / d, 3, 0.5, 1.0, 1e-10, opts=pl.options(mode=mode, comm=comm))
    a1, b1, st1, s1 = pl.plssvm_train_ex(X, y, kernel, 1.0 / d, 3, 0.5, 1.0, 1e-10, opts=pl.options(mode=mode))
    a3, b3, st3, s3 = pl.plssvm_train_ex(X, y, kernel, 1.0 / d, 3, 0.5, 1.0, 1e-10, opts=pl.options(mode=mode))
    p = np.random.default_rng(5).standard_normal(m - 1)
    o1, _ = pl.plssvm_qtilde_matvec(X, p, kernel, 1.0 / d, 3, 0.5, 1.0, opts=pl.options(mode=mode, comm=comm))
    o2, _ = pl.plssvm_qtilde_matvec(X, p, kernel, 1.0 / d, 3, 0.5, 1.0, opts=pl.options(mode=mode, comm=comm))
    o3, _ = pl.plssvm_qtilde_matvec(X, p, kernel, 1.0 / d, 3, 0.5, 1.0, opts=pl.options(mode=mode))
    print(rank, "sharded repeat equal:", np.array_equal(a, a2), s.iterations, s2.iterations,
          "single repeat equal:", np.array_equal(a1, a3), "matvec sharded repeat equal", np.array_equal(o1, o2),
          "sharded vs single matvec", np.abs(o1 - o3).max(), flush=True)
    print(rank, "sharded", st, s.iterations, s.rel_residual, b, "| single", st1, s1.iterations, s1.rel_residual, b1,
          "| dalpha", np.linalg.norm(a - a1) / np.linalg.norm(a1), flush=True)
    pl.plssvm_comm_destroy(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(worker, args=(2, port, int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])), nprocs=2)

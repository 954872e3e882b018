"""Host logic of the row-sharded multi-GPU path (paper_1401_5171_b200/dist.py) on CPU with the gloo
backend, world size 2: row partition, the single all-gather exchange, the fixed rank-order sum
(every rank obtains bitwise the same G and R), status agreement, and the assembled Q.  The step
functions are CPU stand-ins (numpy Gram of the shard, oracle Cholesky / substitution); the GPU
kernels of the same steps are checked in tests/test_gpu_dist_steps.py."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_1401_5171_b200.dist import normal_rows, row_partition

M, N, KA, KZ, SEED = 300, 12, 1e3, 1e2, 31


class CpuSteps:
    def gram_rows(self, Ar, Z, r0, mr):
        A_blk = Ar.numpy()[:, :mr].T            # mr x m
        Zd = Z.numpy()[:, :M].T                 # m x n
        return torch.from_numpy(np.ascontiguousarray((Zd[r0:r0 + mr].T @ (A_blk @ Zd)).T))

    def sum_partials(self, P):
        G = P[0].clone()
        for c in range(1, P.shape[0]):
            G += P[c]
        return G

    def potrf(self, G):
        R, info = oracle.potrf(G.numpy())
        return torch.from_numpy(R), info

    def status(self, info):
        return int(info)

    def trsm_rows(self, Z, R, r0, mr):
        Zr = np.ascontiguousarray(Z.numpy()[:, r0:r0 + mr])
        return torch.from_numpy(oracle.trsm(Zr, R.numpy(), mr))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        parts = row_partition(M, world)
        r0, mr = parts[rank]
        Ar = torch.from_numpy(gen.A_rows(M, KA, SEED, r0, r0 + mr))
        p = gen.problem(M, N, KA, KZ, SEED, with_A=False)
        Q, R, st = normal_rows(Ar, torch.from_numpy(p.Z), r0, mr, steps=CpuSteps())
        np.save(os.path.join(out, f"R{rank}.npy"), R.numpy())
        np.save(os.path.join(out, f"Q{rank}.npy"), Q.numpy())
        with open(os.path.join(out, f"st{rank}"), "w") as f:
            f.write(str(st))
    finally:
        dist.destroy_process_group()


def test_row_partition_covers_and_aligns():
    for m, w in ((300, 2), (40000, 8), (65, 4), (1000, 3)):
        parts = row_partition(m, w)
        assert parts[0][0] == 0 and sum(mr for _, mr in parts) == m
        for (a, ma), (b, _) in zip(parts, parts[1:]):
            assert a + ma == b and b % 64 == 0


def test_two_rank_gloo_matches_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    R0, R1 = np.load(tmp_path / "R0.npy"), np.load(tmp_path / "R1.npy")
    assert np.array_equal(R0, R1)                                  # same bits on every rank
    assert open(tmp_path / "st0").read() == open(tmp_path / "st1").read() == "0"
    # single process with the same steps and the same (rank-order) partial sum
    p = gen.problem(M, N, KA, KZ, SEED)
    steps = CpuSteps()
    Z = torch.from_numpy(p.Z)
    parts = row_partition(M, world)
    Gs = [steps.gram_rows(torch.from_numpy(gen.A_rows(M, KA, SEED, r0, r0 + mr)), Z, r0, mr) for r0, mr in parts]
    G = steps.sum_partials(torch.stack(Gs))
    R, info = steps.potrf(G)
    assert info == 0 and np.array_equal(R.numpy(), R0)
    Q = np.concatenate([np.load(tmp_path / f"Q{r}.npy") for r in range(world)], axis=1)
    Qs = oracle.trsm(p.Z, R.numpy(), M)
    assert np.array_equal(Q, Qs)
    # and the sharded factorisation is CHOLQR of the whole problem (oracle, tolerance)
    Qo, Ro, sto = oracle.normal(p.A, p.Z, M)
    assert sto == 0
    assert np.linalg.norm(R0 - Ro) / np.linalg.norm(Ro) < 1e-12
    assert oracle.componentwise_ratio(p.Z, Q, R0, M) <= oracle.gamma(N + 1)

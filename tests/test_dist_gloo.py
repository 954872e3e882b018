"""Host logic of the row-sharded multi-GPU path (paper_1401_5171_b200/dist.py) on CPU with the gloo
backend: row partition, the all-gather exchanges (one per Cholesky: one for oqr_normal and the
Householder PRE-CHOLQR, two for repeated CHOLQR and the Cholesky-QR PRE-CHOLQR), the fixed
rank-order sums (every rank obtains bitwise the same G and R), status agreement, and the assembled
Q.  The step functions are CPU stand-ins (numpy Grams of the shard, oracle Cholesky / substitution
/ products / Householder QR); the GPU kernels of the same steps are checked in
tests/test_gpu_dist_steps.py and tests/test_gpu_dist_gloo.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_1401_5171_b200.dist import VARIANTS_ROWS, row_partition

M, N, KA, KZ, SEED = 300, 12, 1e3, 1e2, 31


class CpuSteps:
    def __init__(self, m):
        self.m = m

    def gram_rows(self, Ar, Z, r0, mr):
        A_blk = Ar.numpy()[:, :mr].T            # mr x m
        Zd = Z.numpy()[:, :self.m].T            # m x n
        return torch.from_numpy(np.ascontiguousarray((Zd[r0:r0 + mr].T @ (A_blk @ Zd)).T))

    def gram_euclid_rows(self, Z, r0, mr):
        Zr = Z.numpy()[:, r0:r0 + mr].T
        return torch.from_numpy(np.ascontiguousarray((Zr.T @ Zr).T))

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

    def trsm_full(self, Z, R):
        return torch.from_numpy(oracle.trsm(np.ascontiguousarray(Z.numpy()[:, :self.m]), R.numpy(), self.m))

    def trmm(self, R2, R1):
        return torch.from_numpy(oracle.trmm(R2.numpy(), R1.numpy()))

    def hhqr(self, Z):
        Y, S = oracle.hhqr(np.ascontiguousarray(Z.numpy()[:, :self.m]), self.m)
        return torch.from_numpy(Y), torch.from_numpy(S)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out, variant, m, n):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        parts = row_partition(m, world)
        r0, mr = parts[rank]
        Ar = torch.from_numpy(gen.A_rows(m, KA, SEED, r0, r0 + mr))
        p = gen.problem(m, n, KA, KZ, SEED, with_A=False)
        Q, R, st = VARIANTS_ROWS[variant](Ar, torch.from_numpy(p.Z), r0, mr, steps=CpuSteps(m))
        np.save(os.path.join(out, f"R{rank}.npy"), R.numpy())
        np.save(os.path.join(out, f"Q{rank}.npy"), Q.numpy())
        with open(os.path.join(out, f"st{rank}"), "w") as f:
            f.write(str(st))
    finally:
        dist.destroy_process_group()


def test_row_partition_covers_and_aligns():
    for m, w in ((300, 2), (40000, 8), (1000, 3), (65, 4), (200, 8), (1000, 8), (8, 8), (9, 8)):
        parts = row_partition(m, w)
        assert parts[0][0] == 0 and sum(mr for _, mr in parts) == m
        assert all(mr >= 1 for _, mr in parts), (m, w, parts)   # no empty shard (the exchange needs all)
        for (a, ma), (b, _) in zip(parts, parts[1:]):
            assert a + ma == b
        if m >= 64 * w * 2:                                      # aligned when that leaves no rank empty
            assert all(r0 % 64 == 0 for r0, _ in parts), (m, w, parts)
    with pytest.raises(ValueError):
        row_partition(3, 4)


def _single_process(variant, m, n, world):
    """The same steps in one process, partials summed in rank order: the bits the ranks must hold."""
    steps = CpuSteps(m)
    p = gen.problem(m, n, KA, KZ, SEED, with_A=False)
    Z = torch.from_numpy(p.Z)
    parts = row_partition(m, world)
    Ars = [torch.from_numpy(gen.A_rows(m, KA, SEED, r0, r0 + mr)) for r0, mr in parts]

    def chol(Gs):
        R, info = steps.potrf(steps.sum_partials(torch.stack(Gs)))
        assert info == 0
        return R
    if variant == "normal":
        R = chol([steps.gram_rows(Ar, Z, r0, mr) for Ar, (r0, mr) in zip(Ars, parts)])
        return steps.trsm_full(Z, R).numpy(), R.numpy()
    if variant == "normal2":
        R1 = chol([steps.gram_rows(Ar, Z, r0, mr) for Ar, (r0, mr) in zip(Ars, parts)])
        Q1 = steps.trsm_full(Z, R1)
        R2 = chol([steps.gram_rows(Ar, Q1, r0, mr) for Ar, (r0, mr) in zip(Ars, parts)])
        return steps.trsm_full(Q1, R2).numpy(), steps.trmm(R2, R1).numpy()
    if variant == "prequr":
        S = chol([steps.gram_euclid_rows(Z, r0, mr) for r0, mr in parts])
        Y = steps.trsm_full(Z, S)
    else:
        Y, S = steps.hhqr(Z)
    U = chol([steps.gram_rows(Ar, Y, r0, mr) for Ar, (r0, mr) in zip(Ars, parts)])
    return steps.trsm_full(Y, U).numpy(), steps.trmm(U, S).numpy()


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr", "prequr_hh"])
@pytest.mark.parametrize("world,m,n", [(2, M, N), (3, 40, 30)])
def test_gloo_ranks_match_single_process(tmp_path, variant, world, m, n):
    # (3, 40, 30): shards of 13-14 rows < n = 30 columns (the local Gram / substitution blocks
    # are wider than tall), unaligned partition
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), variant, m, n), nprocs=world, join=True)
    Rs = [np.load(tmp_path / f"R{r}.npy") for r in range(world)]
    assert all(np.array_equal(Rs[0], Rr) for Rr in Rs[1:])        # same bits on every rank
    assert all(open(tmp_path / f"st{r}").read() == "0" for r in range(world))
    Q = np.concatenate([np.load(tmp_path / f"Q{r}.npy") for r in range(world)], axis=1)
    Qs, Rsp = _single_process(variant, m, n, world)
    assert np.array_equal(Rsp, Rs[0]) and np.array_equal(Q, Qs)
    # and the sharded factorisation is the variant of the whole problem (oracle, tolerance)
    p = gen.problem(m, n, KA, KZ, SEED)
    Qo, Ro, sto = oracle.VARIANTS[variant](p.A, p.Z, m)
    assert sto == 0
    assert np.linalg.norm(Rs[0] - Ro) / np.linalg.norm(Ro) < 1e-11
    rho = oracle.componentwise_ratio(p.Z, Q, Rs[0], m)
    assert rho <= (oracle.gamma(n + 1) if variant == "normal" else m * n * n * oracle.U)

"""The product row-sharded path (paper_1401_5171_b200/dist.normal_rows with the liboqr kernels) run
by two real ranks of a torch.distributed process group sharing the one GPU of the test box; the
n x n exchange goes through gloo on host copies, so no kernel ever waits on another rank.  Checks:
every rank holds bitwise the same R, the assembled Q and R pass the CHOLQR gates against the
oracle (T2, T5), and R equals the single-process sharded composition bitwise."""
import os
import socket

import numpy as np
import pytest

import gen
import oracle
from oracle import U, gamma

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

M, N, KA, KZ, SEED = 3000, 40, 1e3, 1e2, 33


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out, variant="normal"):
    import torch.distributed as dist
    from paper_1401_5171_b200.dist import VARIANTS_ROWS, row_partition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r0, mr = row_partition(M, world)[rank]
        ldar = mr + (mr & 1)
        Ar = torch.from_numpy(gen.A_rows(M, KA, SEED, r0, r0 + mr, lda=ldar)).cuda()
        p = gen.problem(M, N, KA, KZ, SEED, with_A=False)
        Q, R, st = VARIANTS_ROWS[variant](Ar, torch.from_numpy(p.Z).cuda(), r0, mr)
        torch.cuda.synchronize()
        np.save(os.path.join(out, f"R{rank}.npy"), R.cpu().numpy())
        np.save(os.path.join(out, f"Q{rank}.npy"), Q.cpu().numpy())
        with open(os.path.join(out, f"st{rank}"), "w") as f:
            f.write(str(st))
    finally:
        dist.destroy_process_group()


def test_two_ranks_one_gpu_gloo(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    assert open(tmp_path / "st0").read() == open(tmp_path / "st1").read() == "0"
    R0, R1 = np.load(tmp_path / "R0.npy"), np.load(tmp_path / "R1.npy")
    assert np.array_equal(R0, R1)
    Q = np.concatenate([np.load(tmp_path / f"Q{r}.npy") for r in range(world)], axis=1)
    p = gen.problem(M, N, KA, KZ, SEED)
    assert oracle.componentwise_ratio(p.Z, Q, R0, M) <= gamma(N + 1)
    Qo, Ro, sto = oracle.normal(p.A, p.Z, M)
    E, Eo = oracle.orth_error(p.A, Q, M), oracle.orth_error(p.A, Qo, M)
    normQ = np.linalg.norm(oracle.from_cm(Qo, M), 2)
    assert E <= 10 * Eo + 10 * N * U * float(np.max(p.d)) * normQ ** 2
    # the same shards composed in one process give bitwise the same R
    import paper_1401_5171_b200 as oqr
    from paper_1401_5171_b200.dist import row_partition
    Z = torch.from_numpy(p.Z).cuda()
    Gs = []
    for r0, mr in row_partition(M, world):
        ldar = mr + (mr & 1)
        Gs.append(oqr.gram_rows(torch.from_numpy(gen.A_rows(M, KA, SEED, r0, r0 + mr, lda=ldar)).cuda(), Z, r0, mr))
    R, info = oqr.potrf(oqr.sum_partials(torch.stack(Gs)))
    assert int(info.item()) == 0 and np.array_equal(R.cpu().numpy(), R0)


@pytest.mark.parametrize("variant", ["normal2", "prequr", "prequr_hh"])
def test_two_ranks_one_gpu_gloo_variants(tmp_path, variant):
    """The two-exchange variants (repeated CHOLQR, Cholesky-QR PRE-CHOLQR) and the Householder
    PRE-CHOLQR over two real ranks: same R bits on both, Theorem 3 / oracle-relative gates."""
    import torch.multiprocessing as mp
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), variant), nprocs=world, join=True,
                       start_method="spawn")
    assert open(tmp_path / "st0").read() == open(tmp_path / "st1").read() == "0"
    R0, R1 = np.load(tmp_path / "R0.npy"), np.load(tmp_path / "R1.npy")
    assert np.array_equal(R0, R1)
    Q = np.concatenate([np.load(tmp_path / f"Q{r}.npy") for r in range(world)], axis=1)
    p = gen.problem(M, N, KA, KZ, SEED)
    Qo, Ro, sto = oracle.VARIANTS[variant](p.A, p.Z, M)
    assert sto == 0
    rho, rho_o = oracle.componentwise_ratio(p.Z, Q, R0, M), oracle.componentwise_ratio(p.Z, Qo, Ro, M)
    assert rho <= 10 * rho_o + 4 * gamma(N + 1)
    E, Eo = oracle.orth_error(p.A, Q, M), oracle.orth_error(p.A, Qo, M)
    normQ = np.linalg.norm(oracle.from_cm(Qo, M), 2)
    assert E <= 10 * Eo + 10 * N * U * float(np.max(p.d)) * normQ ** 2

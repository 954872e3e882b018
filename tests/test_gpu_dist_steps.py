"""GPU kernels of the row-sharded path (oqr_gram_rows, oqr_sum_partials, oqr_trsm on row shards) on
ONE device, shards processed one after another (no kernel waits for another), against the oracle:
  * sum of the shard Grams = oqr_gram within 2 gamma_{3m} |Z|^T|A||Z| (T1; bilinearity of
    Algorithm 1 lines 1-2); a single shard covering all rows is bitwise oqr_gram;
  * the assembled Q, R meet the CHOLQR gates T2, T5 against the oracle."""
import numpy as np
import pytest

import gen
import oracle
from oracle import U, gamma

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oqr():
    import paper_1401_5171_b200 as m
    m.lib()
    return m


@pytest.mark.parametrize("m,n,world", [(1000, 40, 2), (4000, 50, 3), (333, 21, 2), (2048, 200, 4)])
def test_row_sharded_cholqr(oqr, m, n, world):
    from paper_1401_5171_b200.dist import row_partition
    ka, kz, seed = 1e3, 1e2, 41
    p = gen.problem(m, n, ka, kz, seed)
    Z = torch.from_numpy(p.Z).cuda()
    parts = row_partition(m, world)
    Gs = []
    for r0, mr in parts:
        ldar = mr + (mr & 1)  # even leading dimension: tensor-TMA path
        Ar = torch.from_numpy(gen.A_rows(m, ka, seed, r0, r0 + mr, lda=ldar)).cuda()
        Gs.append(oqr.gram_rows(Ar, Z, r0, mr))
    G = oqr.sum_partials(torch.stack(Gs)).cpu().numpy().T
    Go = oracle.from_cm(oracle.gram(p.A, p.Z, m), n)
    Zd = np.abs(oracle.from_cm(p.Z, m))
    M = Zd.T @ (np.abs(oracle.from_cm(p.A, m)) @ Zd)
    assert np.all(np.abs(G - Go) <= 2 * gamma(3 * m) * M)
    R, info = oqr.potrf(torch.from_numpy(oracle.to_cm(G)).cuda())
    assert int(info.item()) == 0
    Q = torch.cat([oqr.trsm_rows(Z, R, r0, mr) for r0, mr in parts], dim=1)
    Qg, Rg = Q.cpu().numpy(), R.cpu().numpy()
    assert oracle.componentwise_ratio(p.Z, Qg, Rg, m) <= gamma(n + 1)
    Qo, Ro, sto = oracle.normal(p.A, p.Z, m)
    E, Eo = oracle.orth_error(p.A, Qg, m), oracle.orth_error(p.A, Qo, m)
    normQ = np.linalg.norm(oracle.from_cm(Qo, m), 2)
    assert E <= 10 * Eo + 10 * n * U * float(np.max(p.d)) * normQ ** 2


def test_single_shard_is_bitwise_oqr_gram(oqr):
    p = gen.problem(1000, 30, 1e2, 1e2, 3)
    A = torch.from_numpy(p.A).cuda()
    Z = torch.from_numpy(p.Z).cuda()
    assert torch.equal(oqr.gram_rows(A, Z, 0, 1000), oqr.gram(A, Z))


def test_normal_rows_world1_matches_normal(oqr):
    from paper_1401_5171_b200.dist import normal_rows
    p = gen.problem(700, 33, 1e2, 1e2, 4)
    A = torch.from_numpy(p.A).cuda()
    Z = torch.from_numpy(p.Z).cuda()
    Q1, R1, s1 = normal_rows(A, Z, 0, 700)
    Q2, R2, s2 = oqr.normal(A, Z)
    assert s1 == s2 == 0
    assert torch.equal(R1, R2) and torch.equal(Q1, Q2)


def test_normal_rows_over_a_one_rank_nccl_group(oqr):
    """The exchange step of the row-sharded path (all-gather of the n x n partials in rank order,
    then the fixed-order sum) through NCCL on this GPU: a one-rank group, so no rank waits on
    another; with one shard the result is bitwise oqr_normal's."""
    import socket
    import torch.distributed as dist
    from paper_1401_5171_b200.dist import normal_rows
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        p = gen.problem(1000, 40, 1e3, 1e2, 8)
        A = torch.from_numpy(p.A).cuda()
        Z = torch.from_numpy(p.Z).cuda()
        Q1, R1, s1 = normal_rows(A, Z, 0, 1000)
        Q2, R2, s2 = oqr.normal(A, Z)
        assert s1 == s2 == 0
        assert torch.equal(R1, R2) and torch.equal(Q1, Q2)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant", ["normal", "normal2", "prequr", "prequr_hh"])
def test_rows_variants_world1_bitwise(oqr, variant):
    """With one shard every row-sharded variant runs exactly the single-GPU call's kernels: bitwise
    equal results (repeated CHOLQR and both PRE-CHOLQRs included)."""
    from paper_1401_5171_b200.dist import VARIANTS_ROWS
    p = gen.problem(900, 37, 1e3, 1e3, 5)
    A = torch.from_numpy(p.A).cuda()
    Z = torch.from_numpy(p.Z).cuda()
    Q1, R1, s1 = VARIANTS_ROWS[variant](A, Z, 0, 900)
    Q2, R2, s2 = oqr.VARIANTS[variant](A, Z)
    assert s1 == s2 == 0
    assert torch.equal(R1, R2) and torch.equal(Q1, Q2)


@pytest.mark.parametrize("mr", [1, 5, 17, 39])
def test_wide_row_blocks(oqr, mr):
    """Row blocks with fewer rows than columns (n = 40): the Euclidean Gram of the block and the
    row-wise substitution (oqr_gram_euclid / oqr_trsm accept n > m), against the oracle."""
    m, n, r0 = 300, 40, 101
    p = gen.problem(m, n, 1.0, 1e2, 6, with_A=False)
    Z = torch.from_numpy(p.Z).cuda()
    G = oqr.gram_euclid_rows(Z, r0, mr).cpu().numpy().T
    Zb = oracle.from_cm(p.Z, m)[r0:r0 + mr]
    Go = oracle.from_cm(oracle.gram_euclid(oracle.to_cm(Zb), mr), n)
    assert np.all(np.abs(G - Go) <= 2 * gamma(3 * mr) * (np.abs(Zb).T @ np.abs(Zb)))
    Rs, _ = oracle.potrf(oracle.gram_euclid(p.Z, m))
    Q = oqr.trsm_rows(Z, torch.from_numpy(Rs).cuda(), r0, mr).cpu().numpy()
    Qo = oracle.trsm(oracle.to_cm(Zb), Rs, mr)
    assert oracle.componentwise_ratio(oracle.to_cm(Zb), Q, Rs, mr) <= gamma(n + 1)
    assert np.linalg.norm(Q - Qo) <= 2 * gamma(n + 1) * np.linalg.norm(np.abs(oracle.from_cm(Qo, mr)) @ np.abs(
        oracle.from_cm(Rs, n))) / np.linalg.svd(oracle.from_cm(Rs, n), compute_uv=False)[-1]


def test_trmm_export(oqr):
    rng = np.random.default_rng(9)
    n = 37
    R2, R1 = np.triu(rng.standard_normal((n, n))), np.triu(rng.standard_normal((n, n)))
    R = oqr.trmm(torch.from_numpy(oracle.to_cm(R2)).cuda(), torch.from_numpy(oracle.to_cm(R1)).cuda()).cpu().numpy()
    Ro = oracle.trmm(oracle.to_cm(R2), oracle.to_cm(R1))
    assert np.array_equal(np.tril(oracle.from_cm(R, n), -1), np.zeros((n, n)))
    assert np.all(np.abs(R - Ro) <= 2 * gamma(n) * oracle.to_cm(np.abs(R2) @ np.abs(R1)))

"""Row-sharded multi-GPU oblique QR.

Rank r owns rows R_r = [r0, r0 + mr) of A (an mr x m column-major block) and all of Z.
Algorithm 1 lines 1-2 are bilinear, so G = sum_r Z_{R_r}^T (A_{R_r,:} Z):

    1. G_r = oqr_gram_rows(...)                  local fused Gram kernel (A_r streamed once)
    2. all-gather of the n x n partials          the ONE exchange (8 n^2 bytes per rank), NCCL
    3. G = oqr_sum_partials(gathered)            fixed rank order => bitwise-identical G, R on
                                                 every rank (an all-reduce has no order guarantee)
    4. R = oqr_potrf(G)                          redundantly on every rank (n^3/3 flops)
    5. Q_r = oqr_trsm(Z_{R_r}, R)                local rows

The two-pass variants need one such exchange per Cholesky (the paper's communication-avoiding
property: one reduction per CHOLQR pass):
  * normal2 (repeated CHOLQR, reading R1): pass 1 as above; every rank then forms ALL rows of
    Q1 = Z R1^{-1} (it holds all of Z; m n^2 flops, no exchange) as the B operand of pass 2, whose
    partials Q1_{R_r}^T (A_{R_r,:} Q1) are exchanged once more; Q_r = Q1_{R_r} R2^{-1}, R = R2 R1.
  * prequr (Algorithm 2, Euclidean Cholesky-QR pre-step, reading R2): the Euclidean Gram of the
    local rows Z_{R_r}^T Z_{R_r} is exchanged (first exchange), S = chol, Y = Z S^{-1} on all rows
    of every rank, then the A-stage with the second exchange; R = U S.
  * prequr_hh (Algorithm 2 with the Householder pre-step): the Householder QR of Z runs on every
    rank (all of Z is there; the pre-step is O(m n^2) against the A-stage's 2 m^2 n / N), then the
    A-stage with one exchange; R = U S.
Status codes are the single-GPU ones (first Cholesky k, second n + k) and identical on all ranks.

torch.distributed supplies the collective and the process group (plumbing only); every
arithmetic step is a liboqr kernel.  ``steps`` is injectable so that the host logic (partition,
gather order, fixed-order sum, status agreement) is testable on CPU with the gloo backend
(tests/test_dist_gloo.py); the product path uses :class:`GpuSteps`.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

ALIGN = 64  # row-shard boundaries on panel boundaries of the fused Gram kernel


def row_partition(m: int, world: int, align: int = ALIGN) -> list[tuple[int, int]]:
    """Contiguous row ranges [(r0, mr)] covering 0..m-1, every rank at least one row.  Boundaries
    are multiples of `align` (the fused Gram's 64-row panels) whenever that leaves no rank empty;
    otherwise (m < world * align, roughly) the rows are split evenly without alignment."""
    if m < world:
        raise ValueError(f"row_partition: m = {m} rows cannot give each of {world} ranks a row")
    cuts = [0]
    for k in range(1, world):
        cuts.append(min(m, max(cuts[-1], int(round(k * m / world / align)) * align)))
    cuts.append(m)
    if any(b <= a for a, b in zip(cuts, cuts[1:])):
        cuts = [k * m // world for k in range(world + 1)]
    return [(cuts[k], cuts[k + 1] - cuts[k]) for k in range(world)]


class GpuSteps:
    """The product steps: liboqr kernels on the local GPU."""

    def __init__(self):
        import paper_1401_5171_b200 as oqr
        self.oqr = oqr

    def gram_rows(self, Ar, Z, r0, mr):
        return self.oqr.gram_rows(Ar, Z, r0, mr)

    def gram_euclid_rows(self, Z, r0, mr):
        return self.oqr.gram_euclid_rows(Z, r0, mr)

    def sum_partials(self, P):
        return self.oqr.sum_partials(P)

    def potrf(self, G):
        return self.oqr.potrf(G)

    def status(self, info) -> int:
        return int(info.item())

    def trsm_rows(self, Z, R, r0, mr):
        return self.oqr.trsm_rows(Z, R, r0, mr)

    def trsm_full(self, Z, R):
        return self.oqr.trsm(Z, R, Z.shape[1])

    def trmm(self, R2, R1):
        return self.oqr.trmm(R2, R1)

    def hhqr(self, Z):
        return self.oqr.hhqr(Z, m=Z.shape[1])


def _exchange(G_r, group):
    """All-gather of the n x n partials in rank order (the one collective per Cholesky)."""
    n = G_r.shape[0]
    if not dist.is_initialized():
        return G_r.reshape(1, n, n)
    world = dist.get_world_size(group)
    gathered = torch.empty((world, n, n), dtype=G_r.dtype, device=G_r.device)
    if G_r.is_cuda and dist.get_backend(group) == "gloo":
        # gloo exchanges host tensors: stage the 8 n^2-byte partials through host memory
        host = torch.empty((world, n, n), dtype=G_r.dtype)
        dist.all_gather(list(host.unbind(0)), G_r.cpu(), group=group)
        gathered.copy_(host)
    else:
        dist.all_gather(list(gathered.unbind(0)), G_r.contiguous(), group=group)  # rank order
    return gathered


def _cholesky(steps, G_r, group):
    G = steps.sum_partials(_exchange(G_r, group))
    R, info = steps.potrf(G)
    return R, steps.status(info)


def normal_rows(Ar, Z, r0: int, mr: int, group=None, steps=None):
    """CHOLQR (Algorithm 1) on a row-sharded A.  Returns (Q_r (n, mr), R (n, n), status) on every
    rank; R and status are identical on all ranks; Q_r holds this rank's rows of Q."""
    steps = steps if steps is not None else GpuSteps()
    R, st = _cholesky(steps, steps.gram_rows(Ar, Z, r0, mr), group)
    if st != 0:
        return None, R, st
    return steps.trsm_rows(Z, R, r0, mr), R, 0


def normal2_rows(Ar, Z, r0: int, mr: int, group=None, steps=None):
    """Repeated CHOLQR (reading R1) on a row-sharded A: two exchanges."""
    steps = steps if steps is not None else GpuSteps()
    n = Z.shape[0]
    R1, st = _cholesky(steps, steps.gram_rows(Ar, Z, r0, mr), group)
    if st != 0:
        return None, R1, st
    Q1 = steps.trsm_full(Z, R1)                       # all m rows on every rank (no exchange)
    R2, st = _cholesky(steps, steps.gram_rows(Ar, Q1, r0, mr), group)
    if st != 0:
        return None, R2, n + st
    return steps.trsm_rows(Q1, R2, r0, mr), steps.trmm(R2, R1), 0


def prequr_rows(Ar, Z, r0: int, mr: int, group=None, steps=None):
    """PRE-CHOLQR (Algorithm 2, Euclidean Cholesky-QR pre-step) on a row-sharded A: two exchanges."""
    steps = steps if steps is not None else GpuSteps()
    n = Z.shape[0]
    S, st = _cholesky(steps, steps.gram_euclid_rows(Z, r0, mr), group)
    if st != 0:
        return None, S, st
    Y = steps.trsm_full(Z, S)
    U, st = _cholesky(steps, steps.gram_rows(Ar, Y, r0, mr), group)
    if st != 0:
        return None, U, n + st
    return steps.trsm_rows(Y, U, r0, mr), steps.trmm(U, S), 0


def prequr_hh_rows(Ar, Z, r0: int, mr: int, group=None, steps=None):
    """PRE-CHOLQR with the Householder pre-step (Algorithm 2 as stated) on a row-sharded A:
    the pre-step on every rank, one exchange."""
    steps = steps if steps is not None else GpuSteps()
    n = Z.shape[0]
    Y, S = steps.hhqr(Z)
    U, st = _cholesky(steps, steps.gram_rows(Ar, Y, r0, mr), group)
    if st != 0:
        return None, U, n + st
    return steps.trsm_rows(Y, U, r0, mr), steps.trmm(U, S), 0


VARIANTS_ROWS = {"normal": normal_rows, "normal2": normal2_rows, "prequr": prequr_rows,
                 "prequr_hh": prequr_hh_rows}

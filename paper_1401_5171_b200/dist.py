"""Row-sharded multi-GPU oblique QR.

Rank r owns rows R_r = [r0, r0 + mr) of A (an mr x m column-major block) and all of Z.
Algorithm 1 lines 1-2 are bilinear, so G = sum_r Z_{R_r}^T (A_{R_r,:} Z):

    1. G_r = oqr_gram_rows(...)                  local fused Gram kernel (A_r streamed once)
    2. all-gather of the n x n partials          the ONE exchange (8 n^2 bytes per rank), NCCL
    3. G = oqr_sum_partials(gathered)            fixed rank order => bitwise-identical G, R on
                                                 every rank (an all-reduce has no order guarantee)
    4. R = oqr_potrf(G)                          redundantly on every rank (n^3/3 flops)
    5. Q_r = oqr_trsm(Z_{R_r}, R)                local rows

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
    """Contiguous row ranges [(r0, mr)] covering 0..m-1, boundaries multiples of `align`."""
    cuts = [0]
    for k in range(1, world):
        cuts.append(min(m, max(cuts[-1], int(round(k * m / world / align)) * align)))
    cuts.append(m)
    return [(cuts[k], cuts[k + 1] - cuts[k]) for k in range(world)]


class GpuSteps:
    """The product steps: liboqr kernels on the local GPU."""

    def __init__(self):
        import paper_1401_5171_b200 as oqr
        self.oqr = oqr

    def gram_rows(self, Ar, Z, r0, mr):
        return self.oqr.gram_rows(Ar, Z, r0, mr)

    def sum_partials(self, P):
        return self.oqr.sum_partials(P)

    def potrf(self, G):
        return self.oqr.potrf(G)

    def status(self, info) -> int:
        return int(info.item())

    def trsm_rows(self, Z, R, r0, mr):
        return self.oqr.trsm_rows(Z, R, r0, mr)


def normal_rows(Ar, Z, r0: int, mr: int, group=None, steps=None):
    """CHOLQR (Algorithm 1) on a row-sharded A.  Returns (Q_r (n, mr), R (n, n), status) on every
    rank; R and status are identical on all ranks; Q_r holds this rank's rows of Q."""
    steps = steps if steps is not None else GpuSteps()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    n = Z.shape[0]
    G_r = steps.gram_rows(Ar, Z, r0, mr)
    if dist.is_initialized():  # the exchange step runs whenever there is a group (also world = 1)
        gathered = torch.empty((world, n, n), dtype=G_r.dtype, device=G_r.device)
        if G_r.is_cuda and dist.get_backend(group) == "gloo":
            # gloo exchanges host tensors: stage the 8 n^2-byte partials through host memory
            host = torch.empty((world, n, n), dtype=G_r.dtype)
            dist.all_gather(list(host.unbind(0)), G_r.cpu(), group=group)
            gathered.copy_(host)
        else:
            dist.all_gather(list(gathered.unbind(0)), G_r.contiguous(), group=group)  # rank order
    else:
        gathered = G_r.reshape(1, n, n)
    G = steps.sum_partials(gathered)
    R, info = steps.potrf(G)
    st = steps.status(info)
    if st != 0:
        return None, R, st
    return steps.trsm_rows(Z, R, r0, mr), R, 0

"""Multi-GPU plumbing: join the clique of an initialised torch.distributed
process group (one process per GPU, launched by torchrun).

torch.distributed only carries the 128-byte NCCL id from rank 0 to the other
ranks; the solve's exchanges (halo planes, plane all-gathers, max
reductions) run inside the engine over NCCL on the engine's stream
(csrc/transport.cpp).  See SURVEY.md 8e and DESIGN.md section 8.
"""
from __future__ import annotations

from .api import Context, nccl_unique_id, slab_plan


def share_unique_id(rank: int) -> bytes:
    """Rank 0 makes an NCCL clique id; every rank returns the same 128 bytes
    (broadcast over the default torch.distributed group: gloo or nccl)."""
    import torch.distributed as td

    box = [nccl_unique_id() if rank == 0 else None]
    td.broadcast_object_list(box, src=0)
    uid = box[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("share_unique_id: malformed NCCL id")
    return bytes(uid)


def join_torch_clique(ctx: Context) -> tuple[int, int]:
    """Make `ctx` a rank of the clique formed by the torch.distributed world
    (no-op for a world of one).  Returns (nranks, rank)."""
    import torch.distributed as td

    if not td.is_available() or not td.is_initialized():
        return 1, 0
    n, r = td.get_world_size(), td.get_rank()
    if n > 1:
        ctx.join_nccl(n, r, share_unique_id(r))
    return n, r


def plan_table(n: int, nranks: int, replicate_n: int = 0) -> list[tuple[int, int, int]]:
    """slab_plan of every rank: [(vrep, z0, nz)] (host only)."""
    return [slab_plan(n, nranks, r, replicate_n) for r in range(nranks)]


def check_plan(n: int, nranks: int, replicate_n: int = 0) -> None:
    """The per-rank plans tile every distributed level exactly once and agree
    on the replicated levels (raises AssertionError otherwise)."""
    table = plan_table(n, nranks, replicate_n)
    vreps = {t[0] for t in table}
    assert len(vreps) == 1, "ranks disagree on the replicated levels"
    vrep = vreps.pop()
    N0 = (1 << n) + 1
    for v in range(vrep if nranks > 1 else 1):
        Nv = (1 << (n - v)) + 1
        covered = []
        for r, (_, z0, nz) in enumerate(table):
            last = 1 if r == nranks - 1 else 0
            kb, cnt = z0 >> v, ((nz - last) >> v) + last
            assert cnt >= 2 or nranks == 1, "a z-slab level needs >= 2 planes per rank"
            covered.extend(range(kb, kb + cnt))
        assert covered == list(range(Nv)), f"level {v}: planes not tiled once"
    assert sum(t[2] for t in table) == N0

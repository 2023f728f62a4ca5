"""One large emulated SGEMM over the GPUs of a process group (SURVEY §8(f)
NEXT 3): B and C are split into contiguous column blocks, A is replicated, and
each rank computes its block C[:, n0:n1] = A B[:, n0:n1] with
emu_sgemm_multicast, whose epilogue stores every finished tile into EVERY
rank's C buffer (symmetric-memory peer pointers over NVLink) -- the all-gather
is fused into the GEMM and overlaps the remaining tiles.  Two device-side
barriers across the ranks, both on the stream the GEMM runs on, order each
step: one BEFORE the first remote store (no rank may overwrite a peer's C
while that peer still reads the previous step's result -- write-after-read),
one after the last (every C is complete when the call's work is done).

Host logic only (argument marshalling and the shard plan); the arithmetic runs
in libemusgemm.so.  Without symmetric memory (a single process, or a backend
without peer mappings) the same call computes the local block and all-gathers
it with torch.distributed -- the baseline the fused path replaces, reported as
such by ``ShardedGemm.exchange``.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

__all__ = ["column_shards", "ShardedGemm"]


def column_shards(n: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous, balanced column blocks [n0, n1) of an n-column matrix, one per
    rank (block sizes differ by at most one column; empty blocks when n < world)."""
    if n < 0 or world < 1:
        raise ValueError("n >= 0 and world >= 1 required")
    return [(r * n // world, (r + 1) * n // world) for r in range(world)]


class ShardedGemm:
    """C (m x n, column-major, ldc = m, replicated on every rank) = A (m x k) B (k x n)
    with rank r owning columns column_shards(n, world)[r].

    ``C`` is this rank's full result buffer, a torch tensor of shape (n, m).
    ``__call__(A, B_r, mode)`` takes the replicated A (k, m) and this rank's
    column block B_r (n1 - n0, k), both column-major device tensors.
    """

    def __init__(self, m: int, n: int, k: int, group=None, device=None, fused: Optional[bool] = None,
                 local: Optional[Callable] = None):
        import torch
        import torch.distributed as dist
        self.m, self.n, self.k = m, n, k
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.n0, self.n1 = column_shards(n, self.world)[self.rank]
        self.device = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                                         if torch.cuda.is_available() else torch.device("cpu"))
        self._local = local            # tests: a stand-in for the device call on CPU process groups
        self._hdl = None
        self._ptrs = None
        want_fused = fused if fused is not None else (self.world > 1 and self.device.type == "cuda")
        if want_fused:   # (fused=True at world size 1 exercises the same path on one GPU)
            import torch.distributed._symmetric_memory as symm_mem
            gname = (group or dist.group.WORLD).group_name
            self.C = symm_mem.empty((n, m), dtype=torch.float32, device=self.device)
            self._hdl = symm_mem.rendezvous(self.C, gname)
            self._ptrs = list(self._hdl.buffer_ptrs)
            self.exchange = "fused: emu_sgemm_multicast epilogue stores into every rank's C (symmetric memory)"
        else:
            self.C = torch.empty((n, m), dtype=torch.float32, device=self.device)
            self.exchange = ("none (single rank)" if self.world == 1
                             else "baseline: local block, then torch.distributed all_gather")

    def __call__(self, A, B_r, mode="fp16", stream=None, kblock=0, flags=0) -> None:
        """One step, enqueued on `stream` (a torch.cuda.Stream; default: the
        current stream).  The caller may read C after the step's work on that
        stream; a later step first waits (device barrier) until every rank has
        reached it, i.e. finished whatever it enqueued before on its stream."""
        m, k = self.m, self.k
        n0, n1 = self.n0, self.n1
        if self._ptrs is not None:
            import torch
            import paper_2308_15152_b200 as emu
            dsts = [p + 4 * n0 * m for p in self._ptrs]
            st = stream if stream is not None else torch.cuda.current_stream()
            with torch.cuda.stream(st):
                self._hdl.barrier(channel=0)     # peers are done with their previous C (WAR)
                if n1 > n0:
                    emu.emu_sgemm_multicast(m, n1 - n0, k, 1.0, A, m, B_r, k, dsts, m, mode, st, kblock, flags)
                self._hdl.barrier(channel=1)     # every block has landed in every C
            return
        self._compute_local(A, B_r, self.C[n0:n1], mode, stream, kblock, flags)
        if self.world > 1:
            self._all_gather()

    def _compute_local(self, A, B_r, C_r, mode, stream, kblock, flags):
        if self._local is not None:
            self._local(A, B_r, C_r)
            return
        import paper_2308_15152_b200 as emu
        if self.n1 > self.n0:
            emu.emu_sgemm_multicast(self.m, self.n1 - self.n0, self.k, 1.0, A, self.m, B_r, self.k, [C_r], self.m,
                                    mode, stream, kblock, flags)

    def _all_gather(self):
        import torch
        import torch.distributed as dist
        blocks = column_shards(self.n, self.world)
        width = max(b - a for a, b in blocks)
        buf = torch.zeros((width, self.m), dtype=self.C.dtype, device=self.C.device)
        buf[: self.n1 - self.n0] = self.C[self.n0:self.n1]
        outs = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        for (a, b), o in zip(blocks, outs):
            self.C[a:b] = o[: b - a]

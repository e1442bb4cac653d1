"""Multi-GPU sharding of a simulation batch: one process per GPU, one tally all-reduce.

Sims are independent (batch.py:1-8), so the global sim index range [0, N) is split
into contiguous per-rank shards.  Every per-sim random stream is a pure function of the global sim
index (NATIVE: Philox counter; MT: the sim's own seed; INJECT: its CSR draw range), so the reduced
tallies are bit-identical for any number of ranks -- the GPU analogue of run_batch's worker-count
invariance (batch.py:110-124, tests/test_batch.py:38-42).

The only collective on the success path is ONE SUM all-reduce of the tally vector
(``bbe_tally_len(n)`` u64 counters, < 1 KB for n = 10), enqueued on the kernel's stream right after
it.  The two complement-encoded "first failing sim" fields (include/bbe_sim.h) need a MAX, not a
SUM: each rank keeps its own values, and only when the summed failure counts are non-zero -- the
same on every rank after the SUM -- does ``settle_first_fields`` run a second (MAX) all-reduce.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TALLY_FIELDS = ("wins", "ranks", "perms", "ct", "blocked", "n_div", "n_bad", "first_div", "first_bad")


def shard_range(n_sims: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of rank in world; sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    return n_sims * rank // world, n_sims * (rank + 1) // world


@dataclass
class TallyLayout:
    n: int
    nperm: int

    @classmethod
    def for_n(cls, n: int) -> "TallyLayout":
        import math

        return cls(n, math.factorial(n) if n <= 6 else 0)

    @property
    def ct(self) -> int:
        return self.n + self.n * self.n + self.nperm

    @property
    def length(self) -> int:
        return self.ct + 6

    @property
    def sum_len(self) -> int:
        """Prefix reduced with SUM; the last two fields are reduced with MAX."""
        return self.ct + 4


def reduce_tally(tally, layout: TallyLayout, group=None):
    """One in-place SUM all-reduce of a rank's tally tensor (torch int64; CUDA for NCCL, CPU for gloo).

    Returns this rank's own "first failing sim" fields (a copy taken before the SUM, which garbles
    them in ``tally``); pass it to ``settle_first_fields`` once the tally has been read."""
    import torch.distributed as dist

    own_first = tally[layout.sum_len:].clone()
    dist.all_reduce(tally, op=dist.ReduceOp.SUM, group=group)
    return own_first


def settle_first_fields(tally, own_first, layout: TallyLayout, group=None) -> None:
    """Restore the MAX-reduced "first failing sim" fields after ``reduce_tally``.

    No collective when no rank failed (the summed n_div / n_bad are zero -- identical on every rank,
    so every rank takes the same branch); else one MAX all-reduce of the saved fields."""
    import torch.distributed as dist

    fails = int(tally[layout.ct + 2]) + int(tally[layout.ct + 3])
    if fails == 0:
        tally[layout.sum_len:] = 0
        return
    dist.all_reduce(own_first, op=dist.ReduceOp.MAX, group=group)
    tally[layout.sum_len:] = own_first.to(tally.device)


@dataclass
class Tally:
    wins: np.ndarray
    ranks: np.ndarray
    perms: np.ndarray | None
    competitor_steps: int
    blocked_steps: int
    n_diverged: int
    n_bad_draws: int
    first_diverged: int
    first_bad_draws: int


def decode_tally(t: np.ndarray, layout: TallyLayout) -> Tally:
    t = np.asarray(t).astype(np.uint64)
    n = layout.n

    def first(v):
        v = int(v)
        return -1 if v == 0 else (2**63 - 1) - v

    return Tally(
        wins=t[:n].copy(),
        ranks=t[n:n + n * n].reshape(n, n).copy(),
        perms=t[n + n * n:layout.ct].copy() if layout.nperm else None,
        competitor_steps=int(t[layout.ct]),
        blocked_steps=int(t[layout.ct + 1]),
        n_diverged=int(t[layout.ct + 2]),
        n_bad_draws=int(t[layout.ct + 3]),
        first_diverged=first(t[layout.ct + 4]),
        first_bad_draws=first(t[layout.ct + 5]),
    )


def encode_first(index: int) -> int:
    """Encoding of a failing sim index as stored in the tally: (2^63 - 1) - index, 0 = none."""
    return 0 if index < 0 else (2**63 - 1) - index


def simulate_sharded(state, config, n_sims: int, seed: int = 0, *, group=None, lanes_per_slot: int = 0,
                     mode: str = "native") -> Tally:
    """A batch over all ranks of ``group`` (one GPU per rank, NCCL).

    Each rank simulates its contiguous shard of [0, n_sims) with global sim indices, the device
    tallies are all-reduced, and every rank returns the job total.  mode="native64" (FP64 state) /
    "native" (FP32 state): Philox keyed by ``seed``; mode="mt": sim i replays the reference's stream random.Random(derive_seed(seed, "run", i))
    -- run_batch's seeds (batch.py:117-119), so the total equals the reference's batch tallies.
    """
    import torch
    import torch.distributed as dist

    from .sim import DeviceLauncher, SimDivergedError

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    lo, hi = shard_range(int(n_sims), rank, world)
    launcher = DeviceLauncher(state, config, lanes_per_slot=lanes_per_slot,
                              native_mode=mode if mode in ("native", "native64") else "native")
    layout = TallyLayout.for_n(len(config.competitors))
    assert layout.length == launcher.tally_len
    tally = torch.zeros(layout.length, dtype=torch.int64, device="cuda")
    launcher.launch(tally.data_ptr(), hi - lo, seed, sim_offset=lo,
                    stream=torch.cuda.current_stream().cuda_stream, mode=mode)
    if world > 1:
        own_first = reduce_tally(tally, layout, group)
        host = tally.cpu()
        settle_first_fields(host, own_first, layout, group)  # own_first stays on the collective's device
        out = decode_tally(host.numpy().view(np.uint64), layout)
    else:
        out = decode_tally(tally.cpu().numpy().view(np.uint64), layout)
    if out.n_diverged:
        raise SimDivergedError(out.first_diverged, f"race exceeded tick_limit in sim {out.first_diverged}")
    return out

"""Multi-GPU plumbing: one process per GPU, torch.distributed.

* Single-instance solves (configs 1-3) do not shard: every rank runs an
  independent replica; timings are combined as max over ranks.
* Batched evaluation (config 4) shards the latent batch across ranks (no
  data-path collective); results are all-gathered once (E[B], grad[B x d]).
* The Lipschitz loss (config 5) shards the pairs; one all_reduce(SUM) of the
  per-rank partial sum, divided by the global pair count.

The compute callables are injected so the same code runs over the CUDA library
on B200 ranks and over any callable in CPU (gloo) tests.
"""
from __future__ import annotations

from typing import Callable, Tuple

import numpy as np


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of `total` items for `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard_range: bad world/rank")
    lo = (total * rank) // world
    hi = (total * (rank + 1)) // world
    return lo, hi


def max_over_ranks(value: float, dist=None, device=None) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sharded_lipschitz_loss(partial_sum: Callable[[np.ndarray, np.ndarray], float], Z1: np.ndarray, Z2: np.ndarray,
                           dist=None, device=None) -> float:
    """mean_p |H(z1_p) - H(z2_p)|_F^2 / |z1_p - z2_p|^2 over all ranks' pairs.

    `partial_sum(Z1_local, Z2_local)` returns the sum (not mean) over its pairs."""
    P = Z1.shape[0]
    if P == 0:
        raise ValueError("lipschitz loss: no pairs")
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    lo, hi = shard_range(P, world, rank)
    local = partial_sum(Z1[lo:hi], Z2[lo:hi]) if hi > lo else 0.0
    if world > 1:
        import torch
        t = torch.tensor([local], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        local = float(t.item())
    return local / P


def sharded_eval(eval_fn: Callable[[np.ndarray], Tuple[np.ndarray, np.ndarray]], Z: np.ndarray, dist=None,
                 device=None) -> Tuple[np.ndarray, np.ndarray]:
    """E[B], G[B x d] for a latent batch sharded across ranks, all-gathered."""
    B, r = Z.shape
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    lo, hi = shard_range(B, world, rank)
    E_loc, G_loc = eval_fn(Z[lo:hi]) if hi > lo else (np.zeros(0), np.zeros((0, r)))
    if world == 1:
        return E_loc, G_loc
    import torch
    buf = np.zeros((B, r + 1))
    buf[lo:hi, 0] = E_loc
    buf[lo:hi, 1:] = G_loc
    t = torch.from_numpy(buf).to(device) if device is not None else torch.from_numpy(buf)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)  # disjoint slices: sum == gather
    out = t.cpu().numpy()
    return out[:, 0].copy(), out[:, 1:].copy()

"""Batch-sharded per-example norms + GNS: the host side of SURVEY.md §8(e).

The reference has no distributed runtime (`SPEC.md:9`, `SPEC.md:484`); this
module is the B200 build's one exchange step. The batch shards into
contiguous example blocks, one per process/GPU. Per-example raw norms never
leave their GPU. Per step, every rank all-reduces two buckets:
- `grads`: every layer's batch-summed parameter gradients, e.g. [dgamma | dbeta], fp32;
- `records`: every layer's 4-double record {sum_b raw(p0), sum_b raw(p1),
  ||grad p0||^2, ||grad p1||^2}, fp64 (the layout `gnsb_ln_bwd` writes to its
  `sums` pointer and `gnsb_gns_step` reads).

After the reduce, slots 2 and 3 hold the sum of the LOCAL squared norms,
which is not the squared norm of the sum. They are re-formed from the
reduced gradients. The corrected per-example norm then uses
B_global: corrected = sum_all raw / B_global * B_global^2
(`proj/src/layers.cpp:39-42`).

The GNS step that follows is `DeviceGnsAccumulator.step(records, B_global)`;
`layer_grad_stats` is its host restatement, used for logging (and for the
CPU tests).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from .gns import GradStats


def shard_bounds(B_global: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous example block [b0, b1) of `rank`. Sizes differ by at most one."""
    if B_global < 1:
        raise ValueError("layers: empty batch")
    if not 0 <= rank < world:
        raise ValueError("sharded: rank outside the world")
    return B_global * rank // world, B_global * (rank + 1) // world


class GradBuckets:
    """The per-step exchange buffers for a list of two-parameter layers.

    widths[l] is the parameter length of layer l (D for a LayerNorm). The
    views `grad(l)` = (p0, p1) and `record(l)` point into the two flat
    buckets, so the kernels write straight into what is all-reduced.
    """

    def __init__(self, widths: Sequence[int], device, grad_dtype: torch.dtype = torch.float32):
        self.widths = [int(w) for w in widths]
        self.device = torch.device(device)
        self.grads = torch.zeros(2 * sum(self.widths), dtype=grad_dtype, device=self.device)
        self.records = torch.zeros(len(self.widths), 4, dtype=torch.float64, device=self.device)
        self._views: List[Tuple[torch.Tensor, torch.Tensor]] = []
        off = 0
        for w in self.widths:
            self._views.append((self.grads[off:off + w], self.grads[off + w:off + 2 * w]))
            off += 2 * w

    def __len__(self) -> int:
        return len(self.widths)

    def grad(self, l: int) -> Tuple[torch.Tensor, torch.Tensor]:
        return self._views[l]

    def record(self, l: int) -> torch.Tensor:
        return self.records[l]

    def reduce(self, group=None, sqnorm: Optional[Callable] = None, records: bool = True) -> None:
        """Sum both buckets over the process group, then re-form ||grad||^2
        of every reduced parameter vector into record slots 2 and 3.

        `sqnorm(v, out)` writes the fp64 squared norm of v into the 0-d
        tensor `out`. The default is the device kernel `gnsb_sqnorm`.
        records=False reduces the gradients only (a plain backward without norms).
        """
        if sqnorm is None:
            from .layers import sqnorm as _device_sqnorm

            sqnorm = _device_sqnorm
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.grads, group=group)
            if records:
                dist.all_reduce(self.records, group=group)
        if not records:
            return
        for l, (p0, p1) in enumerate(self._views):
            sqnorm(p0, out=self.records[l, 2])
            sqnorm(p1, out=self.records[l, 3])


def corrected(sum_raw: float, batch: int) -> float:
    """corrected_mean_sqnorm (proj/src/layers.cpp:39-42), B = the GLOBAL batch."""
    b = float(batch)
    return sum_raw / b * (b * b)


def layer_grad_stats(record: Sequence[float], B_global: int) -> GradStats:
    """PerExample GradStats of one layer (proj/src/trainer.cpp:363-378).

    Parameters are visited in the reference's map order (p1 before p0:
    "beta" < "gamma", "bias" < "weight"), as `gns_step_kernel` does.
    """
    r = [float(v) for v in record]
    g_big = 0.0
    g_big += r[3]
    g_big += r[2]
    g_small = 0.0
    g_small += corrected(r[1], B_global)
    g_small += corrected(r[0], B_global)
    return GradStats(g_big, g_small, int(B_global), 1, int(B_global))

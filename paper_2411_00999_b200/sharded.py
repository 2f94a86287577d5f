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
    """The per-step exchange buffers for a list of layers.

    widths[l] is either an int w (a two-parameter layer of width w each: a
    LayerNorm's gamma/beta) or a pair (w0, w1): a linear layer is (K*L, L),
    a bias-less layer (K*L, 0), an embedding (V*D, 0). The views
    `grad(l)` = (p0, p1) and `record(l)` point into the two flat buckets, so
    the kernels write straight into what is exchanged.

    `reduce()` is the step's ONE collective: on CUDA buckets it runs the C
    ABI's exchange (gnsb_exchange_pack -> one all-reduce of a single fp64
    buffer holding every record and gradient -> gnsb_exchange_unpack, which
    re-forms the squared norms of the reduced gradients).
    """

    def __init__(self, widths: Sequence, device, grad_dtype: torch.dtype = torch.float32):
        self.pairs = [(int(w), int(w)) if isinstance(w, (int,)) or not hasattr(w, "__len__") else
                      (int(w[0]), int(w[1])) for w in widths]
        self.widths = [p0 for p0, _ in self.pairs]
        self.device = torch.device(device)
        self.grads = torch.zeros(sum(a + b for a, b in self.pairs), dtype=grad_dtype, device=self.device)
        self.records = torch.zeros(len(self.pairs), 4, dtype=torch.float64, device=self.device)
        self._views: List[Tuple[torch.Tensor, torch.Tensor]] = []
        off = 0
        for a, b in self.pairs:
            self._views.append((self.grads[off:off + a], self.grads[off + a:off + a + b]))
            off += a + b
        self._ws = None
        self._w2 = None

    def __len__(self) -> int:
        return len(self.pairs)

    def grad(self, l: int) -> Tuple[torch.Tensor, torch.Tensor]:
        return self._views[l]

    def record(self, l: int) -> torch.Tensor:
        return self.records[l]

    # ------------------------------------------------------------ device path
    def _c_args(self):
        import ctypes

        from . import _lib

        if self._w2 is None:
            flat = [v for p in self.pairs for v in p]
            self._w2 = (ctypes.c_int64 * len(flat))(*flat)
            n = ctypes.c_size_t()
            _lib.check(_lib.lib().gnsb_exchange_workspace_size(self._w2, len(self.pairs), ctypes.byref(n)))
            self._ws = torch.zeros(n.value, dtype=torch.uint8, device=self.device)
        dt = {torch.float32: _lib.GNSB_F32, torch.float64: _lib.GNSB_F64}[self.grads.dtype]
        return _lib, dt

    def packed(self, records: bool = True) -> torch.Tensor:
        """fp64 view of the packed exchange buffer (what the collective sums)."""
        self._c_args()
        n = (4 * len(self.pairs) if records else 0) + self.grads.numel()
        return self._ws[: 8 * n].view(torch.float64)

    def pack(self, records: bool = True, stream=None) -> None:
        _lib, dt = self._c_args()
        sp = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        _lib.check(_lib.lib().gnsb_exchange_pack(self.grads.data_ptr(), dt, self._w2, len(self.pairs),
                                                 self.records.data_ptr() if records else None, self._ws.data_ptr(),
                                                 self._ws.numel(), sp))

    def unpack(self, records: bool = True, stream=None) -> None:
        _lib, dt = self._c_args()
        sp = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        _lib.check(_lib.lib().gnsb_exchange_unpack(self.grads.data_ptr(), dt, self._w2, len(self.pairs),
                                                   self.records.data_ptr() if records else None,
                                                   self._ws.data_ptr(), self._ws.numel(), sp))

    def allreduce_nccl(self, comm, records: bool = True, stream=None) -> None:
        """pack -> ncclAllReduce on `comm` (a C-ABI communicator, NcclComm) -> unpack,
        in one stream-ordered C-ABI call (capturable in a CUDA graph)."""
        _lib, dt = self._c_args()
        sp = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        _lib.check(_lib.lib().gnsb_allreduce_buckets(self.grads.data_ptr(), dt, self._w2, len(self.pairs),
                                                     self.records.data_ptr() if records else None,
                                                     self._ws.data_ptr(), self._ws.numel(),
                                                     comm.handle if comm is not None else None, sp))

    def reduce(self, group=None, sqnorm: Optional[Callable] = None, records: bool = True, comm=None) -> None:
        """Sum both buckets over the ranks in ONE collective, then re-form
        ||grad||^2 of every reduced parameter vector into record slots 2 and 3.

        CUDA buckets: with `comm` (NcclComm) the whole exchange is one C-ABI
        call; otherwise pack -> torch.distributed all_reduce of the packed fp64
        buffer over `group` -> unpack.
        `sqnorm(v, out)` (tests on CPU buckets only) restates the exchange with
        torch ops around the same single all-reduce.
        records=False exchanges the gradients only (a plain backward without norms).
        """
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
        if sqnorm is None:
            if self.device.type != "cuda":
                raise RuntimeError("sharded: the exchange runs on CUDA buckets (pass sqnorm= for host tests)")
            if comm is not None:
                self.allreduce_nccl(comm, records)
                return
            self.pack(records)
            if multi:
                dist.all_reduce(self.packed(records), group=group)
            self.unpack(records)
            return
        # host restatement (tests): same layout, same single collective
        nrec = 4 * len(self.pairs) if records else 0
        packed = torch.empty(nrec + self.grads.numel(), dtype=torch.float64, device=self.device)
        if records:
            packed[:nrec] = self.records.reshape(-1)
        packed[nrec:] = self.grads.double()
        if multi:
            dist.all_reduce(packed, group=group)
        self.grads.copy_(packed[nrec:])
        if not records:
            return
        self.records[:, :2] = packed[:nrec].view(-1, 4)[:, :2]
        red = packed[nrec:]
        off = 0
        for l, (a, b) in enumerate(self.pairs):
            sqnorm(red[off:off + a], out=self.records[l, 2])
            sqnorm(red[off + a:off + a + b], out=self.records[l, 3])
            off += a + b


class NcclComm:
    """An NCCL communicator made through the C ABI (gnsb_nccl_*), so that
    gnsb_allreduce_buckets can run the exchange inside a CUDA graph.  The
    unique id travels over the already-initialised torch.distributed group."""

    def __init__(self, group=None):
        import ctypes

        from . import _lib

        lib = _lib.lib()
        if not lib.gnsb_nccl_available():
            raise RuntimeError("nccl: libnccl.so.2 not found")
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _lib.check(lib.gnsb_nccl_get_unique_id(uid))
        t = torch.tensor(list(uid.raw), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0, group=group)
        uid = ctypes.create_string_buffer(bytes(t.cpu().tolist()), 128)
        h = ctypes.c_void_p()
        _lib.check(lib.gnsb_nccl_comm_init_rank(ctypes.byref(h), world, uid, rank))
        self.handle = h
        self.world = world

    def close(self):
        from . import _lib

        if self.handle is not None:
            _lib.check(_lib.lib().gnsb_nccl_comm_destroy(self.handle))
            self.handle = None


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

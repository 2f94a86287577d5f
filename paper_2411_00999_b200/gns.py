"""GNS estimators, mirroring gnstk's gns API (proj/include/gnstk/gns.hpp:16-74).

Host functions call libgnsb's C implementations (same arithmetic, same error
conditions and "gns: ..." messages as proj/src/gns.cpp:14-89).
`DeviceGnsAccumulator` is the device-side accumulator: one single-CTA kernel
per step turns per-layer norm records (written by the fused backward kernels)
into the per-group {g2, s, EMA B_simple} of Trainer::step
(proj/src/trainer.cpp:363-415) without a host round trip.
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import Dict, List, Optional, Sequence

import torch

from . import _lib

LAYER_TYPES = {"embedding": _lib.LAYER_EMBEDDING, "linear": _lib.LAYER_LINEAR, "layernorm": _lib.LAYER_LAYERNORM}
GROUPS = ("total", "embedding", "linear", "layernorm")


@dataclasses.dataclass
class GradStats:
    """gnstk::GradStats (gns.hpp:16-22)."""

    g_big_sqnorm: float = 0.0
    g_small_sqnorm_mean: float = 0.0
    b_big: int = 0
    b_small: int = 0
    n_small: int = 1

    def _c(self) -> _lib.GradStats:
        return _lib.GradStats(self.g_big_sqnorm, self.g_small_sqnorm_mean, self.b_big, self.b_small, self.n_small)


@dataclasses.dataclass
class GnsEstimate:
    g2: float = 0.0
    s: float = 0.0
    b_simple: float = 0.0
    b_simple_defined: bool = False


@dataclasses.dataclass
class EmaState:
    alpha: float = 1.0
    value: float = 0.0
    count: int = 0


def estimate_g2(stats: GradStats) -> float:
    """(B_big |G_big|^2 - B_small |G_small|^2) / (B_big - B_small) (gns.cpp:31-36)."""
    out = ctypes.c_double()
    _lib.check(_lib.lib().gnsb_estimate_g2(ctypes.byref(stats._c()), ctypes.byref(out)))
    return out.value


def estimate_s(stats: GradStats) -> float:
    """(|G_small|^2 - |G_big|^2) / (1/B_small - 1/B_big) (gns.cpp:38-43)."""
    out = ctypes.c_double()
    _lib.check(_lib.lib().gnsb_estimate_s(ctypes.byref(stats._c()), ctypes.byref(out)))
    return out.value


def make_gns_estimate(g2: float, s: float) -> GnsEstimate:
    e = _lib.GnsEstimate()
    _lib.lib().gnsb_make_gns_estimate(g2, s, ctypes.byref(e))
    return GnsEstimate(e.g2, e.s, e.b_simple, bool(e.b_simple_defined))


def ema_update(state: EmaState, x: float) -> EmaState:
    st = _lib.EmaState(state.alpha, state.value, state.count)
    _lib.check(_lib.lib().gnsb_ema_update(ctypes.byref(st), x))
    return EmaState(st.alpha, st.value, st.count)


def smoothed_gns(g2_ema: EmaState, s_ema: EmaState) -> GnsEstimate:
    a = _lib.EmaState(g2_ema.alpha, g2_ema.value, g2_ema.count)
    b = _lib.EmaState(s_ema.alpha, s_ema.value, s_ema.count)
    e = _lib.GnsEstimate()
    _lib.check(_lib.lib().gnsb_smoothed_gns(ctypes.byref(a), ctypes.byref(b), ctypes.byref(e)))
    return GnsEstimate(e.g2, e.s, e.b_simple, bool(e.b_simple_defined))


def aggregate(stats_by_layer: Dict[tuple, GradStats], group: Optional[str]) -> GradStats:
    """gnstk::aggregate (gns.cpp:71-89).  Keys are (name, type) LayerKeys; they
    are visited in LayerKey order (name, then type) like std::map."""
    keys = sorted(stats_by_layer, key=lambda k: (k[0], LAYER_TYPES[k[1]]))
    n = len(keys)
    arr = (_lib.GradStats * max(n, 1))(*[stats_by_layer[k]._c() for k in keys])
    types = (ctypes.c_int32 * max(n, 1))(*[LAYER_TYPES[k[1]] for k in keys])
    out = _lib.GradStats()
    grp = -1 if group is None else LAYER_TYPES[group]
    _lib.check(_lib.lib().gnsb_aggregate(arr, types, n, grp, ctypes.byref(out)))
    return GradStats(out.g_big_sqnorm, out.g_small_sqnorm_mean, out.b_big, out.b_small, out.n_small)


class DeviceGnsAccumulator:
    """Device-side PerExample GNS accumulator (trainer.cpp:324-325, 363-415).

    `step(records, B)` takes a [n_layers, 4] fp64 device tensor of per-layer
    records {sum raw p0, sum raw p1, ||grad p0||^2, ||grad p1||^2} in LayerKey
    order and returns device tensors: groups [4, 4] {g2_raw, s_raw, gns_ema,
    defined} for (total, embedding, linear, layernorm) and layers [n, 2].
    """

    def __init__(self, layer_types: Sequence[str], alpha: float, device):
        self.device = torch.device(device)
        self.types = (ctypes.c_int32 * len(layer_types))(*[LAYER_TYPES[t] for t in layer_types])
        self.n = len(layer_types)
        self.alpha = float(alpha)
        # 8 x gnsb_ema_state {double alpha, double value, int64 count} = 24 bytes each
        self.state = torch.zeros(8 * 3, dtype=torch.float64, device=self.device)
        self.groups = torch.empty(4, 4, dtype=torch.float64, device=self.device)
        self.layers = torch.empty(self.n, 2, dtype=torch.float64, device=self.device)

    def step(self, records: torch.Tensor, B: int):
        assert records.dtype == torch.float64 and records.is_contiguous() and records.shape == (self.n, 4)
        _lib.check(
            _lib.lib().gnsb_gns_step(
                records.data_ptr(), self.types, self.n, int(B), self.alpha, self.state.data_ptr(),
                self.groups.data_ptr(), self.layers.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream,
            )
        )
        return self.groups, self.layers

"""B200-native fused LayerNorm backward + per-example gradient norms + GNS.

A from-scratch sm_100a implementation of the hot path of arXiv 2411.00999 as
exposed by the reference C++ library gnstk (/root/reference/proj):
layernorm_forward / layernorm_backward_simultaneous, the per-example norm
paths for linear layers, and the GNS estimators.  All compute lives in
lib/libgnsb.so (CUDA kernels + the C ABI of include/gnsb.h); this package is
the ctypes host binding that mirrors the reference interface.
"""
from . import _lib
from .layers import (
    LayerGradOutput,
    LayerNormBackwardResult,
    LayerNormCache,
    LayerNormForwardResult,
    LayerNormLayer,
    layernorm_backward_simultaneous,
    layernorm_forward,
    ln_bwd_geometry,
    sqnorm,
    synth_linear,
    synth_ln,
)
from .embedding import embedding_backward_simultaneous, embedding_forward
from .nn import GnsTracker, LayerNormPE
from .model import EmbeddingPE, LinearPE, ToyModelPE
from .linear import (LinearBackwardResult, LinearLayer, linear_backward_simultaneous, linear_forward,
                     linear_perexample_sqnorm_frobenius)
from .gns import (
    DeviceGnsAccumulator,
    EmaState,
    GnsEstimate,
    GradStats,
    aggregate,
    ema_update,
    estimate_g2,
    estimate_s,
    make_gns_estimate,
    smoothed_gns,
)

__all__ = [
    "LayerGradOutput", "LayerNormBackwardResult", "LayerNormCache", "LayerNormForwardResult", "LayerNormLayer",
    "layernorm_backward_simultaneous", "layernorm_forward", "ln_bwd_geometry", "sqnorm", "synth_linear", "synth_ln",
    "DeviceGnsAccumulator", "EmaState", "GnsEstimate", "GradStats", "aggregate", "ema_update", "estimate_g2",
    "estimate_s", "make_gns_estimate", "smoothed_gns", "LinearBackwardResult", "LinearLayer",
    "linear_backward_simultaneous", "linear_perexample_sqnorm_frobenius", "GnsTracker", "LayerNormPE", "EmbeddingPE", "LinearPE", "ToyModelPE",
    "embedding_backward_simultaneous", "embedding_forward", "linear_forward",
]

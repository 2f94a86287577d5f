"""GNS-logged training loop on the GPU kernels.

The PerExample path of the reference trainer (proj/include/gnstk/trainer.hpp,
proj/src/trainer.cpp): every step draws `scheduled_batch` sequences from the
MarkovDataset stream, runs the toy model's forward and backward on the B200
kernels (every instrumented layer's backward also yields its per-example
squared gradient norms), turns the per-layer norm records into GNS statistics
on the device (GnsTracker: groups total / embedding / linear / layernorm, EMA)
and applies SGD or Adam.  With `dtype=torch.float64` and the reference's
initialisation the step logs follow the reference trainer's
(tests/golden/trainer_cases.json); fp32 is the fast configuration.

Only EstimationKind::PerExample exists here: the Microbatch / Subbatch modes,
the JSON config files, the temperature scenarios and the simulator are the
reference's experiment harness, outside the kernel path.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import torch

from .data import MarkovDataset
from .model import ToyModelPE
from .nn import GnsTracker


def _fail(msg: str):
    raise ValueError("trainer: " + msg)


@dataclasses.dataclass
class ScheduleSpec:
    """trainer.hpp:19-27: Fixed(b) or LinearRamp(b_start -> b_end over ramp_tokens)."""

    kind: str = "fixed"  # "fixed" | "linear_ramp"
    b: int = 1
    b_start: int = 1
    b_end: int = 1
    ramp_tokens: int = 1


def scheduled_batch(spec: ScheduleSpec, tokens_processed: int) -> int:
    """trainer.cpp:25-32: round-half-up interpolation with a floor of 1."""
    if spec.kind == "fixed":
        return spec.b
    frac = min(float(tokens_processed) / float(spec.ramp_tokens), 1.0)
    b = float(spec.b_start) + (float(spec.b_end) - float(spec.b_start)) * frac
    r = math.floor(b + 0.5)
    return 1 if r < 1.0 else int(r)


@dataclasses.dataclass
class OptimizerConfig:
    kind: str = "adam"  # "sgd" | "adam"
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


@dataclasses.dataclass
class LrSchedule:
    kind: str = "constant"  # "constant" | "cosine"
    min_ratio: float = 0.1


@dataclasses.dataclass
class TrainConfig:
    """trainer.hpp:59-75 (PerExample estimation only)."""

    vocab: int = 16
    model_dim: int = 32
    hidden_multiplier: int = 2
    n_blocks: int = 2
    seq_len: int = 16
    total_tokens: int = 1 << 18
    optimizer: OptimizerConfig = dataclasses.field(default_factory=OptimizerConfig)
    learning_rate: float = 3e-3
    lr_schedule: LrSchedule = dataclasses.field(default_factory=LrSchedule)
    batch_schedule: ScheduleSpec = dataclasses.field(default_factory=ScheduleSpec)
    ema_alpha: float = 0.02
    seed: int = 1
    loss_scale: float = 1.0


def validate(cfg: TrainConfig) -> None:
    """trainer.cpp:34-60 (the fields this trainer has)."""
    if cfg.vocab < 2:
        _fail("vocab must be >= 2")
    if cfg.model_dim < 2:
        _fail("model_dim must be >= 2")
    if cfg.hidden_multiplier < 1:
        _fail("hidden_multiplier must be >= 1")
    if cfg.n_blocks < 1:
        _fail("n_blocks must be >= 1")
    if cfg.seq_len < 1:
        _fail("seq_len must be >= 1")
    if cfg.total_tokens < 1:
        _fail("total_tokens must be >= 1")
    if cfg.learning_rate < 0.0:
        _fail("learning_rate must be >= 0")
    if not cfg.ema_alpha > 0.0 or cfg.ema_alpha > 1.0:
        _fail("ema_alpha must be in (0, 1]")
    if cfg.loss_scale <= 0.0:
        _fail("loss_scale must be positive")
    if cfg.lr_schedule.kind == "cosine" and not 0.0 <= cfg.lr_schedule.min_ratio <= 1.0:
        _fail("lr min_ratio must be in [0, 1]")
    if cfg.lr_schedule.kind not in ("constant", "cosine"):
        _fail("unknown lr schedule")
    if cfg.optimizer.kind not in ("sgd", "adam"):
        _fail("unknown optimizer")
    bs = cfg.batch_schedule
    if bs.kind == "fixed":
        if bs.b < 1:
            _fail("batch size must be >= 1")
    elif bs.kind == "linear_ramp":
        if bs.b_start < 1 or bs.b_end < bs.b_start:
            _fail("ramp requires 1 <= b_start <= b_end")
        if bs.ramp_tokens < 1:
            _fail("ramp_tokens must be >= 1")
        if bs.ramp_tokens > cfg.total_tokens:
            _fail("ramp_tokens must not exceed total_tokens")
    else:
        _fail("unknown batch schedule")


@dataclasses.dataclass
class GroupLog:
    g2_raw: float = 0.0
    s_raw: float = 0.0
    gns_ema: float = 0.0
    gns_defined: bool = False


@dataclasses.dataclass
class PerLayerLog:
    name: str
    type: str
    g2_raw: float
    s_raw: float


@dataclasses.dataclass
class StepLog:
    step: int = 0
    tokens: int = 0  # processed including this step
    batch_size: int = 0
    loss: float = 0.0
    total: GroupLog = dataclasses.field(default_factory=GroupLog)
    embedding: GroupLog = dataclasses.field(default_factory=GroupLog)
    linear: GroupLog = dataclasses.field(default_factory=GroupLog)
    layernorm: GroupLog = dataclasses.field(default_factory=GroupLog)
    layers: List[PerLayerLog] = dataclasses.field(default_factory=list)


class TrainingDiverged(RuntimeError):
    pass


_TYPE_ORDER = {"embedding": 0, "linear": 1, "layernorm": 2}  # LayerType enum order (gns.hpp:42)


class Trainer:
    """trainer.hpp:113-150 / trainer.cpp:234-426, PerExample, on one GPU."""

    def __init__(self, cfg: TrainConfig, device=None, dtype=torch.float64):
        validate(cfg)
        self.cfg = cfg
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self.data = MarkovDataset(cfg.vocab, cfg.seed)
        self.model = ToyModelPE(cfg.vocab, cfg.model_dim, cfg.hidden_multiplier, cfg.n_blocks, seed=cfg.seed,
                                device=self.device, dtype=dtype, init="reference")
        # std::map<LayerKey> order (gns.hpp:42-55): the aggregate sums g_big /
        # g_small over layers in (name, type) order, as gns.cpp:71-89 does
        self.layers = sorted(self.model.instrumented_layers(), key=lambda nm: (nm[0], _TYPE_ORDER[nm[1].layer_type]))
        self.tracker = GnsTracker([m for _, m in self.layers], alpha=cfg.ema_alpha)
        self.step_index = 0
        self.tokens = 0
        self._adam = {}
        self._adam_t = 0

    def done(self) -> bool:
        return self.tokens >= self.cfg.total_tokens

    def current_lr(self) -> float:
        """trainer.cpp:243-249."""
        c = self.cfg
        if c.lr_schedule.kind == "constant":
            return c.learning_rate
        frac = min(float(self.tokens) / float(c.total_tokens), 1.0)
        w = 0.5 * (1.0 + math.cos(3.14159265358979323846 * frac))
        return c.learning_rate * (c.lr_schedule.min_ratio + (1.0 - c.lr_schedule.min_ratio) * w)

    @torch.no_grad()
    def _apply_update(self, lr: float) -> None:
        """trainer.cpp:251-282 (elementwise updates in the parameter dtype)."""
        params = [p for p in self.model.parameters()]
        if self.cfg.optimizer.kind == "sgd":
            for p in params:
                p.sub_(p.grad, alpha=lr)
            return
        o = self.cfg.optimizer
        self._adam_t += 1
        bc1 = 1.0 - math.pow(o.beta1, float(self._adam_t))
        bc2 = 1.0 - math.pow(o.beta2, float(self._adam_t))
        for p in params:
            st = self._adam.get(id(p))
            if st is None:
                st = self._adam[id(p)] = (torch.zeros_like(p), torch.zeros_like(p))
            m, v = st
            g = p.grad
            m.mul_(o.beta1).add_(g, alpha=1.0 - o.beta1)
            v.mul_(o.beta2).add_(g * g, alpha=1.0 - o.beta2)
            p.sub_(lr * (m / bc1) / (torch.sqrt(v / bc2) + o.eps))

    def step(self) -> StepLog:
        """trainer.cpp:284-426, EstimationKind::PerExample."""
        c = self.cfg
        b = scheduled_batch(c.batch_schedule, self.tokens)
        t = c.seq_len
        if b < 2:
            _fail("per-example estimation needs batch size >= 2")
        seqs = [self.data.fill_sequence(t + 1) for _ in range(b)]
        host = torch.tensor(seqs, dtype=torch.int32)
        ids = host[:, :t].contiguous().to(self.device, non_blocking=True)
        targets = host[:, 1:].contiguous().to(self.device, non_blocking=True)
        for p in self.model.parameters():
            p.grad = None
        # model_backward (model.cpp:144-188) on the library kernels
        loss = self.model.forward_backward(ids, targets, c.loss_scale)
        groups, per_layer = self.tracker.step()
        loss_v = float(loss)
        if not math.isfinite(loss_v):
            raise TrainingDiverged(f"trainer: loss diverged at step {self.step_index}")
        g = groups.cpu().tolist()
        pl = per_layer.cpu().tolist()
        log = StepLog(step=self.step_index, batch_size=b, loss=loss_v)
        for i, name in enumerate(("total", "embedding", "linear", "layernorm")):
            setattr(log, name, GroupLog(g[i][0], g[i][1], g[i][2], bool(g[i][3] != 0.0)))
        rows = [PerLayerLog(n, m.layer_type, pl[i][0], pl[i][1]) for i, (n, m) in enumerate(self.layers)]
        log.layers = rows  # already in std::map<LayerKey> order
        self._apply_update(self.current_lr())
        self.tokens += b * t
        self.step_index += 1
        log.tokens = self.tokens
        return log

    def run(self) -> List[StepLog]:
        logs = []
        while not self.done():
            logs.append(self.step())
        return logs

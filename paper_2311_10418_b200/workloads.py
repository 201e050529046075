"""BASELINE.json's five planning configurations, as exact inputs.

Every config uses the reference's own generator (load_dataset, workload.cpp:50-63,
seed 7; FLANv2-like lognormal lengths, workload.h:46-53 defaults) and grid
(ProfileGrid::synthetic with default SyntheticGridParams and axes), the model
ModelConfig::uniform(C, 2, 1024, encdec), Recompute::None and D = 1
(SURVEY.md §8d).  Multi-mini-batch workloads slice one dataset of n*M samples
into consecutive fixed-count mini-batches, so mini-batch 0 of any M equals the
single-mini-batch config.

The K -> t_max_interval mapping and the frozen I / cap are documented in
configs.py (mapping A').
"""
from __future__ import annotations

import numpy as np

from . import capi

from .configs import CONFIGS, INPUT_DIST, SEED, T5_TARGET_DIST, Config  # noqa: F401


def grid() -> capi.Grid:
    return capi.synthetic_grid()


def model(cfg: Config) -> capi.Model:
    return capi.Model.uniform(cfg.stages, 2, cfg.encdec, recompute=0)


def kind_layouts(cfg: Config) -> int:
    """(distinct stage layout, kind with layers) pairs one slice is priced
    over: stages with equal layouts are deduplicated (capi.cu upload_grid)."""
    m = model(cfg)
    lay = {(int(e), int(d)) for e, d in zip(m.encoder_layers, m.decoder_layers) if e > 0 or d > 0}
    return sum((e > 0) + (d > 0) for e, d in lay)


def dataset(cfg: Config, n_minibatches: int | None = None) -> np.ndarray:
    """(n * M, 3) int64 samples (id, input_len, target_len)."""
    m = cfg.minibatches if n_minibatches is None else n_minibatches
    return capi.synthetic_dataset(cfg.n * m, cfg.max_seq_len, SEED, INPUT_DIST,
                                  T5_TARGET_DIST if cfg.encdec else None)


def seg_offsets(cfg: Config, n_minibatches: int) -> np.ndarray:
    return np.arange(n_minibatches + 1, dtype=np.int64) * cfg.n

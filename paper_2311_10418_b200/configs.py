"""BASELINE.json's five planning configurations as plain data (no native
library import: the reference arm of bench.py builds its inputs from these
through the reference's own API, oracle/bind.py).  workloads.py turns them
into inputs through this library.

The reference has no candidate-count knob, only t_max_interval; "K candidates"
maps to I = T_capmax / K (mapping A').  The exact I and cap are
frozen below (derived by tools/derive_configs.py with the C restatement).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

LOGNORMAL = 0  # LengthFamily::Lognormal (workload.h)

SEED = 7
INPUT_DIST = (LOGNORMAL, 5.0, 1.5, 1, 1, 0.8)     # workload.h:46-53 defaults
T5_TARGET_DIST = (LOGNORMAL, 3.5, 1.2, 1, 1, 0.8)


@dataclass(frozen=True)
class Config:
    name: str
    desc: str
    encdec: bool
    n: int              # samples per mini-batch
    stages: int         # pipeline stages C (model and DpOptions::stage_count)
    K: int              # t_max candidates (via mapping A')
    max_seq_len: int
    minibatches: int = 1
    cap_mult: float = 0.0        # cap = cap_mult * max singleton act_mem (0: +inf)
    interval: float = math.nan   # frozen I (exact)
    mem_cap: float = math.inf    # frozen cap (exact)


CONFIGS = {
    "C1": Config("C1", "GPT cost model, 256-seq mini-batch, 4 stages, 32 t_max candidates",
                 False, 256, 4, 32, 8192,
                 interval=float.fromhex("0x1.875f6fd21ff2fp+19")),    # 801531.4944
    "C2": Config("C2", "T5 encoder-decoder, 1024 seqs/mini-batch, 8 stages, 64 t_max candidates",
                 True, 1024, 8, 64, 8192,
                 interval=float.fromhex("0x1.875f6fd21ff2fp+20")),    # 1603062.9888
    "C3": Config("C3", "GPT 8192 seqs/mini-batch, 16 stages, activation-memory limit binding, "
                 "128 t_max candidates", False, 8192, 16, 128, 8192, cap_mult=4.0,
                 interval=float.fromhex("0x1.875f6fd21ff2fp+11"),     # 3130.9824
                 mem_cap=float.fromhex("0x1.47ae147ae147bp+10")),     # 1310.72
    # C (stages) and K for C4/C5 are not given by BASELINE.json; assumed as in SURVEY.md §8d.
    "C4": Config("C4", "Whole-epoch planning: 4096 independent 2048-seq mini-batches",
                 False, 2048, 8, 64, 8192, minibatches=4096,
                 interval=float.fromhex("0x1.875f6fd21ff2fp+21")),    # 3206125.9776 (mini-batch 0)
    "C5": Config("C5", "Long-tail stress: 65536 seqs truncated at 65536 tokens, T5, 256 t_max",
                 True, 65536, 8, 256, 65536,
                 # no cap: T_capmax = slice [0, n) (monotone grid), / 256
                 interval=float.fromhex("0x1.442c3c9eecbfcp+30")),    # 1359679271.7312
}

"""Seeded synthetic inputs shared by the oracle tests, the parity tests and bench.py.

This package holds none of the method's arithmetic: only graph/stream
generation (numpy in ``gen.py``; the bit-identical CUDA generator in
``csrc/gen.cu`` bound by ``gpu.py``) and the five BASELINE.json configs.
"""
from dataclasses import dataclass

from . import gen  # noqa: F401


@dataclass(frozen=True)
class Config:
    name: str
    kind: str            # "er" | "grid" | "rmat" | "incr"
    seed: int
    scale: int = 0       # rmat / incr
    rows: int = 0        # grid
    cols: int = 0
    n_batches: int = 0   # incr
    n_ins: int = 0
    n_q: int = 0


# BASELINE.json configs[0..4]; seed = config number
C1 = Config("C1-er-100k", "er", 1)
C2 = Config("C2-grid-4096", "grid", 2, rows=4096, cols=4096)
C3 = Config("C3-rmat-24", "rmat", 3, scale=24)
C4 = Config("C4-rmat-27", "rmat", 4, scale=27)
# 2^28 ops in 2^20-op batches, 90 % inserts: floor(0.9 * 2^20) = 943,718 (reading R16)
C5 = Config("C5-incr-2^26", "incr", 5, scale=26, n_batches=256, n_ins=943_718, n_q=104_858)
CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}
BY_INDEX = {1: C1, 2: C2, 3: C3, 4: C4, 5: C5}

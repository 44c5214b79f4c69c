"""Schedule knobs of the reference runtime (graphlets/parallel.py:32-51).

The GPU entry points accept a ``ParallelConfig`` for signature
compatibility and validate it exactly like the reference, but results never
depend on it (the reference contract is schedule invariance,
parallel.py:7-9): the device grid, degree binning and on-device work
cursors replace fork workers, batch claiming and the fixed-order merge.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

from .errors import GraphletError

MAX_BATCH_SIZE = 4096


class WorkerFailure(GraphletError):
    """Kept for API parity; the device path never forks workers."""


@dataclass(frozen=True)
class ParallelConfig:
    workers: int | None = None
    batch_size: int = 64
    ordering: str = "input"

    def __post_init__(self):
        if self.workers is not None and self.workers < 1:
            raise ValueError("workers must be >= 1")
        if not 1 <= self.batch_size <= MAX_BATCH_SIZE:
            raise ValueError(f"batch_size must be in [1, {MAX_BATCH_SIZE}]")
        if self.ordering not in ("input", "degree-desc"):
            raise ValueError("ordering must be 'input' or 'degree-desc'")

    def resolved_workers(self) -> int:
        return self.workers if self.workers is not None else (os.cpu_count() or 1)

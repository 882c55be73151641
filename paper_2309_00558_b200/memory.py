"""Per-model GPU memory costs (host-side description only).

The accounting itself -- footprint in resident-insertion order and the
admission test -- runs inside the device placement kernel
(csrc/gs_kernel.cuh ``footprint`` / ``admit``, csrc/gs_xlh.cuh ``xl_footprint``), restating
pkg/src/gshare_sim/memory_model.py:61-88.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import ValidationError

#: Default per-GPU capacity in MB (reference: memory_model.py:18).
DEFAULT_GPU_MEMORY_MB = 16384.0


@dataclass(frozen=True)
class MemorySpec:
    """MB costs of one model: private copy, shared-runtime share, server share."""

    mem_noshare_mb: float
    mem_runtime_mb: float
    mem_server_mb: float

    def __post_init__(self):
        for label in ("mem_noshare_mb", "mem_runtime_mb", "mem_server_mb"):
            value = getattr(self, label)
            ok = isinstance(value, (int, float)) and math.isfinite(value) and value > 0
            if not ok:
                raise ValidationError(
                    f"{label} must be a positive finite number, got {value!r}")


DEFAULT_MEMORY_SPEC = MemorySpec(mem_noshare_mb=1200.0, mem_runtime_mb=900.0,
                                 mem_server_mb=600.0)

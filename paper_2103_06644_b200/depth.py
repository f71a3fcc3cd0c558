"""``DepthImage`` -- the reference's organized depth lattice (``synth.py:69-114``).

A host-side value type (fp64 metres + validity), kept so that reference callers can pass
the same objects.  Every fitting entry point of this package uploads it to the device:
``values`` as fp64 (``RF_DEPTH_F64_M``) and ``valid`` as the uint8 mask.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MM_PER_METER = 1000.0


@dataclass
class DepthImage:
    """Depth in metres with a validity mask; invalid pixels are excluded from every sum."""

    values: np.ndarray
    valid: np.ndarray = field(default=None)  # type: ignore[assignment]

    def __post_init__(self) -> None:
        self.values = np.asarray(self.values, dtype=np.float64)
        if self.values.ndim != 2:
            raise ValueError(f"depth lattice must be 2D, got shape {self.values.shape}")
        positive = np.isfinite(self.values) & (self.values > 0)
        if self.valid is None:
            self.valid = positive
        else:
            self.valid = np.asarray(self.valid, dtype=bool)
            if self.valid.shape != self.values.shape:
                raise ValueError(f"mask shape {self.valid.shape} != depth shape {self.values.shape}")
            self.valid = self.valid & positive

    @property
    def height(self) -> int:
        return self.values.shape[0]

    @property
    def width(self) -> int:
        return self.values.shape[1]

    def to_millimeters(self) -> np.ndarray:
        """Quantize to uint16 millimetres, 0 marking invalid pixels (synth.py:100-105)."""
        mm = np.where(self.valid, np.round(self.values * MM_PER_METER), 0.0)
        if np.any(mm > np.iinfo(np.uint16).max):
            raise ValueError("depth exceeds uint16 millimeter range")
        return mm.astype(np.uint16)

    @classmethod
    def from_millimeters(cls, mm: np.ndarray) -> "DepthImage":
        mm = np.asarray(mm)
        return cls(values=mm.astype(np.float64) / MM_PER_METER, valid=mm > 0)

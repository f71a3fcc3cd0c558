"""Host-side depth frame type with the reference's validity contract (``synth.py:69-114``).

The GPU kernels apply the same rule on the device (``primary_of`` in
``csrc/rf_tile_kernel.cuh``): a sample takes part in a fit iff it is finite, strictly positive
and not masked out; uint16 millimetres convert as ``mm / 1000.0``.  This module keeps that rule
available on the host so reference callers can hand the same objects to ``fit_rect`` /
``segment``; every fitting entry point uploads ``values`` as fp64 (``RF_DEPTH_F64_M``) and
``valid`` as the uint8 mask.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MM_PER_METER = 1000.0
_U16_MAX = float(np.iinfo(np.uint16).max)


def _as_lattice(values) -> np.ndarray:
    lat = np.asarray(values, dtype=np.float64)
    if lat.ndim != 2:
        raise ValueError(f"depth lattice must be 2D, got shape {lat.shape}")
    return lat


def _validity(lat: np.ndarray, mask) -> np.ndarray:
    """Finite, positive samples, further restricted by an optional caller mask."""
    usable = np.isfinite(lat)
    usable &= lat > 0
    if mask is None:
        return usable
    m = np.asarray(mask, dtype=bool)
    if m.shape != lat.shape:
        raise ValueError(f"mask shape {m.shape} != depth shape {lat.shape}")
    return usable & m


@dataclass
class DepthImage:
    """Depth lattice in metres (fp64) with the mask of samples that enter the fits."""

    values: np.ndarray
    valid: np.ndarray = field(default=None)  # type: ignore[assignment]

    def __post_init__(self) -> None:
        self.values = _as_lattice(self.values)
        self.valid = _validity(self.values, self.valid)

    @property
    def height(self) -> int:
        return int(self.values.shape[0])

    @property
    def width(self) -> int:
        return int(self.values.shape[1])

    def to_millimeters(self) -> np.ndarray:
        """uint16 millimetres, round half to even; 0 marks invalid samples."""
        scaled = np.rint(self.values * MM_PER_METER)
        scaled[~self.valid] = 0.0
        if scaled.size and scaled.max() > _U16_MAX:
            raise ValueError("depth exceeds uint16 millimeter range")
        return scaled.astype(np.uint16)

    @classmethod
    def from_millimeters(cls, mm: np.ndarray) -> "DepthImage":
        raw = np.asarray(mm)
        return cls(values=raw.astype(np.float64) / MM_PER_METER, valid=raw > 0)

"""The reference's integral backend on the device (drop-in for ``rangefit.integral``).

Names, fields and errors follow ``/root/reference/pkg/src/rangefit/integral.py``:
``Rect``, ``IntegralImage``, ``ChannelStack``, ``build_integral``, ``box_sum``,
``build_constant_channels``, ``build_standard_implicit_channels``,
``build_rgbd_implicit_channels``, ``build_standard_explicit_channels``,
``build_rgbd_explicit_channels`` and the channel-name constants (``integral.py:36-47``).

Every table is a device ``float64`` tensor ``[H+1, W+1]`` built by ``rf_build_channel`` /
``rf_integral`` (``csrc/rf_integral.cu``): the channel value with the reference's fp64
expression, masked to 0, summed down each column and then along each row in numpy's order
-- the tables equal the reference's bit for bit.  Box sums run on the device
(``rf_box_sums``).  The per-pixel hot path does not use these tables (its window sums are
tile-local); they serve reference callers of the integral API.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterable

import numpy as np
import torch

from . import _native as N
from .depth import DepthImage
from .fitting import Rect
from .pixels import TanAngleMaps

CONSTANT_CHANNELS = ("tx2", "txty", "ty2", "tx", "ty")
STANDARD_IMPLICIT_CHANNELS = ("x2", "xy", "xz", "x", "y2", "yz", "y", "z2", "z")
RGBD_IMPLICIT_CHANNELS = ("tx_over_z", "ty_over_z", "inv_z", "inv_z2")
STANDARD_EXPLICIT_CHANNELS = ("x2", "xy", "x", "y2", "y", "xz", "yz", "z")
RGBD_EXPLICIT_CHANNELS = ("tx_over_z", "ty_over_z", "inv_z")
HOLE_CORRECTION_CHANNELS = ("m_tx2", "m_txty", "m_ty2", "m_tx", "m_ty")
COUNT_CHANNEL = "count"


@dataclass(frozen=True)
class IntegralImage:
    """Summed-area table with a zero first row and column (integral.py:69-86); device fp64."""

    name: str
    table: torch.Tensor

    @property
    def height(self) -> int:
        return self.table.shape[0] - 1

    @property
    def width(self) -> int:
        return self.table.shape[1] - 1


@dataclass(frozen=True)
class ChannelStack:
    """Named integral images sharing one validity-count channel (integral.py:89-128)."""

    channels: dict
    count: IntegralImage
    scatter_names: tuple
    constant: bool = False
    residual_name: str | None = None
    hole_corrected: bool = False

    def __post_init__(self) -> None:
        shape = tuple(self.count.table.shape)
        for ch in self.channels.values():
            if tuple(ch.table.shape) != shape:
                raise ValueError(f"channel {ch.name!r} shape {tuple(ch.table.shape)} != count shape {shape}")

    @property
    def height(self) -> int:
        return self.count.height

    @property
    def width(self) -> int:
        return self.count.width

    def per_frame_channel_names(self) -> tuple:
        """Every depth-dependent channel in the stack (excludes the count)."""
        return tuple(self.channels.keys())


def _check_rect(rect, width: int, height: int) -> None:
    r = Rect(*rect)
    if not (0 <= r.x0 <= r.x1 <= width and 0 <= r.y0 <= r.y1 <= height):
        raise ValueError(f"rect {r} out of bounds for {width}x{height} image")


def _stream(device: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def build_integral(channel, mask=None, name: str = "", device=None) -> IntegralImage:
    """Single-pass summed-area table of an arbitrary 2-D channel (integral.py:136-149)."""
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    c = torch.as_tensor(np.asarray(channel) if not isinstance(channel, torch.Tensor) else channel)
    if c.dim() != 2:
        raise ValueError(f"channel must be 2D, got shape {tuple(c.shape)}")
    c = c.to(device=dev, dtype=torch.float64).contiguous()
    mptr = None
    if mask is not None:
        m = torch.as_tensor(np.asarray(mask) if not isinstance(mask, torch.Tensor) else mask)
        if tuple(m.shape) != tuple(c.shape):
            raise ValueError(f"mask shape {tuple(m.shape)} != channel shape {tuple(c.shape)}")
        m = m.to(device=dev, dtype=torch.uint8).contiguous()
        mptr = m.data_ptr()
    H, W = c.shape
    table = torch.empty((H + 1, W + 1), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        N.check(N.load().rf_integral(c.data_ptr(), W, mptr, H, W, table.data_ptr(), _stream(dev)), "build_integral")
    return IntegralImage(name=name, table=table)


def box_sums(tables, rects) -> np.ndarray:
    """Box sums of several same-shape tables over many rects in one launch -> [nrects, ntables]."""
    tables = list(tables)
    if not tables:
        return np.zeros((len(rects), 0))
    if len(tables) > N.RF_MAX_BOX_CHANNELS:
        raise ValueError(f"at most {N.RF_MAX_BOX_CHANNELS} tables per call")
    dev = tables[0].device
    H, W = tables[0].shape[0] - 1, tables[0].shape[1] - 1
    rr = np.asarray([(0, *tuple(r)) for r in rects], dtype=np.int32).reshape(-1, 5)
    for r in rr:
        _check_rect(r[1:], W, H)
    d_rects = torch.from_numpy(rr).to(dev)
    out = torch.empty((len(rr), len(tables)), dtype=torch.float64, device=dev)
    ptrs = (ctypes.c_void_p * len(tables))(*[t.data_ptr() for t in tables])
    with torch.cuda.device(dev):
        N.check(N.load().rf_box_sums(ptrs, len(tables), H, W, d_rects.data_ptr(), len(rr), out.data_ptr(),
                                     _stream(dev)), "box_sums")
    return out.cpu().numpy()


def box_sum(integral: IntegralImage, rect) -> float:
    """Sum of the source channel over rect via the 4-lookup identity (integral.py:152-158)."""
    _check_rect(rect, integral.width, integral.height)
    return float(box_sums([integral.table], [rect])[0, 0])


class _DeviceDepth:
    """One depth frame on the device for rf_build_channel."""

    def __init__(self, depth, maps: TanAngleMaps):
        dev = torch.device("cuda", maps.device)
        self.mask = None
        if isinstance(depth, DepthImage):
            if (depth.height, depth.width) != (maps.height, maps.width):
                raise ValueError(f"depth {depth.width}x{depth.height} does not match "
                                 f"maps {maps.width}x{maps.height}")
            self.values = torch.from_numpy(np.ascontiguousarray(depth.values)).to(dev)
            self.mask = torch.from_numpy(np.ascontiguousarray(depth.valid, dtype=np.uint8)).to(dev)
            self.dtype = N.RF_DEPTH_F64_M
            self.all_valid = bool(depth.valid.all())
        else:
            t = depth if isinstance(depth, torch.Tensor) else torch.as_tensor(np.asarray(depth))
            if t.dim() != 2:
                raise ValueError(f"depth lattice must be 2D, got shape {tuple(t.shape)}")
            if tuple(t.shape) != (maps.height, maps.width):
                raise ValueError(f"depth {t.shape[1]}x{t.shape[0]} does not match maps {maps.width}x{maps.height}")
            if t.dtype == torch.float64:
                self.dtype = N.RF_DEPTH_F64_M
            elif t.dtype == torch.float32:
                self.dtype = N.RF_DEPTH_F32_M
            elif t.dtype in (torch.uint16, torch.int16):
                self.dtype = N.RF_DEPTH_U16_MM
            else:
                raise ValueError(f"unsupported depth dtype {t.dtype}")
            self.values = t.to(dev).contiguous()
            self.all_valid = None  # read from the count table
        self.device = dev


def _table(maps: TanAngleMaps, name: str, depth: _DeviceDepth | None) -> IntegralImage:
    dev = torch.device("cuda", maps.device)
    table = torch.empty((maps.height + 1, maps.width + 1), dtype=torch.float64, device=dev)
    st = N.load().rf_build_channel(maps.handle, depth.values.data_ptr() if depth else None,
                                   depth.dtype if depth else 0, maps.width,
                                   depth.mask.data_ptr() if depth is not None and depth.mask is not None else None,
                                   N.RF_CHANNELS[name], table.data_ptr(), _stream(dev))
    N.check(st, f"build channel {name}")
    return IntegralImage(name=name, table=table)


def _frame_stack(depth, maps: TanAngleMaps, names: Iterable[str], scatter_names, residual_name=None,
                 hole_channels: bool = False) -> ChannelStack:
    d = _DeviceDepth(depth, maps)
    count = _table(maps, COUNT_CHANNEL, d)
    channels = {name: _table(maps, name, d) for name in names}
    hole_corrected = False
    if hole_channels:
        all_valid = d.all_valid
        if all_valid is None:
            all_valid = float(count.table[-1, -1].item()) == maps.width * maps.height
        hole_corrected = not all_valid
        if hole_corrected:
            channels.update({name: _table(maps, name, d) for name in HOLE_CORRECTION_CHANNELS})
    return ChannelStack(channels=channels, count=count, scatter_names=tuple(scatter_names), constant=False,
                        residual_name=residual_name, hole_corrected=hole_corrected)


def build_constant_channels(maps: TanAngleMaps) -> ChannelStack:
    """Camera-constant tables tan_x^2, tan_x tan_y, tan_y^2, tan_x, tan_y; the count counts
    every pixel (integral.py:188-199)."""
    channels = {name: _table(maps, name, None) for name in CONSTANT_CHANNELS}
    count = _table(maps, "ones", None)
    count = IntegralImage(name=COUNT_CHANNEL, table=count.table)
    return ChannelStack(channels=channels, count=count, scatter_names=CONSTANT_CHANNELS, constant=True)


def build_standard_implicit_channels(depth, maps: TanAngleMaps) -> ChannelStack:
    """Per-frame tables of X^2, XY, XZ, X, Y^2, YZ, Y, Z^2, Z (integral.py:217-237)."""
    return _frame_stack(depth, maps, STANDARD_IMPLICIT_CHANNELS, STANDARD_IMPLICIT_CHANNELS)


def build_rgbd_implicit_channels(depth, maps: TanAngleMaps) -> ChannelStack:
    """Per-frame tables of tan_x/Z, tan_y/Z, 1/Z, 1/Z^2, plus the masked tan monomials when
    the frame has invalid pixels (integral.py:240-263)."""
    return _frame_stack(depth, maps, RGBD_IMPLICIT_CHANNELS, RGBD_IMPLICIT_CHANNELS, hole_channels=True)


def build_standard_explicit_channels(depth, maps: TanAngleMaps, include_residual: bool = True) -> ChannelStack:
    """Per-frame tables of the standard explicit normal equations (+ Z^2) (integral.py:266-295)."""
    names = STANDARD_EXPLICIT_CHANNELS + (("z2",) if include_residual else ())
    return _frame_stack(depth, maps, names, STANDARD_EXPLICIT_CHANNELS,
                        residual_name="z2" if include_residual else None)


def build_rgbd_explicit_channels(depth, maps: TanAngleMaps, include_residual: bool = True) -> ChannelStack:
    """Per-frame tables tan_x/Z, tan_y/Z, 1/Z (+ 1/Z^2), plus the masked tan monomials when
    the frame has invalid pixels (integral.py:298-325)."""
    names = RGBD_EXPLICIT_CHANNELS + (("inv_z2",) if include_residual else ())
    return _frame_stack(depth, maps, names, RGBD_EXPLICIT_CHANNELS,
                        residual_name="inv_z2" if include_residual else None, hole_channels=True)

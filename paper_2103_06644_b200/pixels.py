"""Host side of the per-pixel path: camera tables and the batched ``fit_pixels``.

Mirrors the reference's fitting vocabulary (``rangefit``):

* :class:`CameraIntrinsics` -- reference ``camera.py:35-75`` (same fields and
  validation; non-zero ``delta_x``/``delta_y`` lattices take the tiled lattice kernel).
* :func:`compute_tan_maps` -- reference ``camera.py:124-135``; here it builds
  the per-camera device tables (``rf_tables_create``) once.
* :class:`HostPipeline` -- host frames in, host outputs out, copies overlapped with the
  kernels (the reference-facing call with host buffers).
* :func:`fit_pixels` -- the batched per-pixel entry the reference lacks (all four
  reference formulations, ``FORMULATIONS``, ``fitting.py:45-49``): for
  every pixel it is ``fit_rect(depth, maps, Rect(max(x-r,0), max(y-r,0),
  min(x+r+1,W), min(y+r+1,H)), formulation, backend)`` (``fitting.py:757-786``)
  followed by the A18 output convention of SURVEY.md: unit normal, offset,
  ``rms_residual``, curvature and a status byte.  Per-pixel failures become
  status bits, never exceptions; argument errors raise ``ValueError`` like the
  reference.

Everything runs through ``librangefit_b200.so``; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N

IMPLICIT_STANDARD = "implicit-standard"
IMPLICIT_RGBD = "implicit-rgbd"
EXPLICIT_STANDARD = "explicit-standard"
EXPLICIT_RGBD = "explicit-rgbd"
# reference FORMULATIONS order (fitting.py:49); ids index rf_fit_pixels' output array
FORMULATIONS = (IMPLICIT_STANDARD, IMPLICIT_RGBD, EXPLICIT_STANDARD, EXPLICIT_RGBD)
PIXEL_FORMULATIONS = (IMPLICIT_STANDARD, IMPLICIT_RGBD)  # the headline pair (north_star)
MIN_SAMPLES = {IMPLICIT_STANDARD: 4, IMPLICIT_RGBD: 4, EXPLICIT_STANDARD: 3, EXPLICIT_RGBD: 3}
_FORM_ID = {f: i for i, f in enumerate(FORMULATIONS)}

STATUS_INPUT_VALID = N.RF_PIX_INPUT_VALID
STATUS_FIT = N.RF_PIX_FIT
STATUS_DEGENERATE = N.RF_PIX_DEGENERATE


@dataclass(frozen=True)
class CameraIntrinsics:
    """Pinhole parameters (reference ``camera.py:35-75``)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    delta_x: np.ndarray | None = None
    delta_y: np.ndarray | None = None

    def __post_init__(self) -> None:
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError(f"focal lengths must be positive, got ({self.fx}, {self.fy})")
        if self.width <= 0 or self.height <= 0:
            raise ValueError(f"image size must be positive, got {self.width}x{self.height}")
        if not (0 <= self.cx < self.width and 0 <= self.cy < self.height):
            raise ValueError(
                f"principal point ({self.cx}, {self.cy}) outside {self.width}x{self.height} image"
            )
        for name in ("delta_x", "delta_y"):
            lattice = getattr(self, name)
            if lattice is None:
                lattice = np.zeros((self.height, self.width))
            else:
                lattice = np.asarray(lattice, dtype=np.float64)
                if lattice.shape != (self.height, self.width):
                    raise ValueError(
                        f"{name} shape {lattice.shape} does not match image ({self.height}, {self.width})"
                    )
            object.__setattr__(self, name, lattice)


@dataclass
class TanAngleMaps:
    """Per-camera device tables (reference ``TanAngleMaps``, ``camera.py:78-96``).

    The lattices are separable (``tan_x`` depends on the column only, ``tan_y``
    on the row only), so the device holds W + H float64 values.
    """

    intrinsics: CameraIntrinsics
    device: int
    _handle: ctypes.c_void_p = field(repr=False)

    @property
    def width(self) -> int:
        return self.intrinsics.width

    @property
    def height(self) -> int:
        return self.intrinsics.height

    @property
    def tan_x(self) -> np.ndarray:
        """The reference's (H, W) lattice ``(x + delta_x - cx) / fx`` (camera.py:131-134), the
        same values the device tables hold (one row when delta = 0, the lattice otherwise)."""
        i = self.intrinsics
        return (np.arange(i.width, dtype=np.float64)[None, :] + i.delta_x - i.cx) / i.fx

    @property
    def tan_y(self) -> np.ndarray:
        """The reference's (H, W) lattice ``(y + delta_y - cy) / fy`` (camera.py:131-134)."""
        i = self.intrinsics
        return (np.arange(i.height, dtype=np.float64)[:, None] + i.delta_y - i.cy) / i.fy

    @property
    def handle(self) -> ctypes.c_void_p:
        if not self._handle:
            raise ValueError("camera tables were released")
        return self._handle

    def release(self) -> None:
        if self._handle:
            N.load().rf_tables_destroy(self._handle)
            self._handle = ctypes.c_void_p()

    def __del__(self) -> None:  # pragma: no cover - interpreter shutdown order
        try:
            self.release()
        except Exception:
            pass


def compute_tan_maps(intrinsics: CameraIntrinsics, device: int | torch.device | None = None) -> TanAngleMaps:
    """Build the device tan tables once per camera (``camera.py:124-135``)."""
    if device is None:
        device = torch.cuda.current_device()
    if isinstance(device, torch.device):
        device = device.index if device.index is not None else torch.cuda.current_device()
    lib = N.load()
    intr = N.RfIntrinsics(intrinsics.fx, intrinsics.fy, intrinsics.cx, intrinsics.cy,
                          intrinsics.width, intrinsics.height)
    dx = np.ascontiguousarray(intrinsics.delta_x, dtype=np.float64)
    dy = np.ascontiguousarray(intrinsics.delta_y, dtype=np.float64)
    handle = ctypes.c_void_p()
    st = lib.rf_tables_create(ctypes.byref(intr), dx.ctypes.data, dy.ctypes.data, int(device),
                              ctypes.byref(handle))
    N.check(st, "compute_tan_maps")
    return TanAngleMaps(intrinsics=intrinsics, device=int(device), _handle=handle)


@dataclass
class PixelFits:
    """Per-pixel outputs of one formulation, each ``[B, H, W]`` (normal ``[B, H, W, 3]``)."""

    normal: torch.Tensor
    offset: torch.Tensor
    residual: torch.Tensor
    curvature: torch.Tensor
    status: torch.Tensor

    @staticmethod
    def empty(batch: int, height: int, width: int, device) -> "PixelFits":
        f = dict(dtype=torch.float32, device=device)
        return PixelFits(
            normal=torch.empty((batch, height, width, 3), **f),
            offset=torch.empty((batch, height, width), **f),
            residual=torch.empty((batch, height, width), **f),
            curvature=torch.empty((batch, height, width), **f),
            status=torch.empty((batch, height, width), dtype=torch.uint8, device=device),
        )

    def _c(self, batch: int, height: int, width: int, device: torch.device) -> N.RfPixelOut:
        """C view of caller-provided output planes, after checking that the kernels can write a
        [batch, height, width] result into them (shape, element type, device, contiguity)."""
        shape = (batch, height, width)
        for name, t, dt, sh in (("normal", self.normal, torch.float32, shape + (3,)),
                                ("offset", self.offset, torch.float32, shape),
                                ("residual", self.residual, torch.float32, shape),
                                ("curvature", self.curvature, torch.float32, shape),
                                ("status", self.status, torch.uint8, shape)):
            ok_shape = tuple(t.shape) == sh or (batch == 1 and tuple(t.shape) == sh[1:])  # [H, W] frame
            if not ok_shape or t.dtype != dt:
                raise ValueError(f"output {name} must be {dt} of shape {sh}, got {t.dtype} {tuple(t.shape)}")
            if t.device != device:
                raise ValueError(f"output {name} on {t.device}, depth on {device}")
            if not t.is_contiguous():
                raise ValueError("output tensors must be contiguous")
        return N.RfPixelOut(self.normal.data_ptr(), self.offset.data_ptr(), self.residual.data_ptr(),
                            self.curvature.data_ptr(), self.status.data_ptr())

    @property
    def fit_mask(self) -> torch.Tensor:
        return (self.status & STATUS_FIT) != 0


def _depth_dtype(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return N.RF_DEPTH_F32_M
    if t.dtype == torch.float64:
        return N.RF_DEPTH_F64_M
    if t.dtype in (torch.uint16, torch.int16):
        return N.RF_DEPTH_U16_MM
    raise ValueError(f"depth must be float32/float64 metres or uint16 millimetres, got {t.dtype}")


def fit_pixels(
    depth: torch.Tensor,
    maps: TanAngleMaps,
    window: int,
    formulations=PIXEL_FORMULATIONS,
    mask: torch.Tensor | None = None,
    out: dict | None = None,
    stream: torch.cuda.Stream | None = None,
) -> dict:
    """Fit a plane over the (2r+1)-square window around every pixel.

    ``depth``: CUDA tensor ``[B, H, W]`` or ``[H, W]``, float32 metres or uint16
    millimetres (converted on device as ``mm / 1000.0``, reference
    ``synth.py:111-114``).  Rows may be padded (``depth.stride(-2) >= W``); the
    last dimension must be contiguous.  Returns ``{formulation: PixelFits}``.
    The launch is asynchronous on ``stream`` (default: torch's current stream).
    """
    if isinstance(formulations, str):
        formulations = (formulations,)
    formulations = tuple(formulations)
    for f in formulations:
        if f not in _FORM_ID:
            raise ValueError(f"unknown formulation {f!r}; expected one of {FORMULATIONS}")
    if not isinstance(depth, torch.Tensor) or not depth.is_cuda:
        raise ValueError("depth must be a CUDA tensor (the sm_100a path has no CPU fallback)")
    squeeze = depth.dim() == 2
    d = depth.unsqueeze(0) if squeeze else depth
    if d.dim() != 3:
        raise ValueError(f"depth must be [B, H, W] or [H, W], got shape {tuple(depth.shape)}")
    B, H, W = d.shape
    if (H, W) != (maps.height, maps.width):
        raise ValueError(f"depth {W}x{H} does not match maps {maps.width}x{maps.height}")
    temps = []  # tensors this call creates on the current stream and the kernel reads on `stream`
    if d.stride(-1) != 1 or (B > 1 and d.stride(0) != d.stride(1) * H):
        d = d.contiguous()
        temps.append(d)
    dtype = _depth_dtype(d)
    if d.device.index != maps.device:
        raise ValueError(f"depth on cuda:{d.device.index} but maps on cuda:{maps.device}")
    if window < 1 or window % 2 == 0:
        raise ValueError(f"window must be a positive odd integer, got {window}")
    mptr = None
    if mask is not None:
        m = mask.unsqueeze(0) if mask.dim() == 2 else mask
        if tuple(m.shape) != (B, H, W):
            raise ValueError(f"mask shape {tuple(mask.shape)} != depth shape {tuple(depth.shape)}")
        m2 = m.to(device=d.device, dtype=torch.uint8).contiguous()
        if m2.data_ptr() != m.data_ptr():
            temps.append(m2)
        m = m2
        mptr = m.data_ptr()
    if out is None:
        out = {f: PixelFits.empty(B, H, W, d.device) for f in formulations}
        temps += [getattr(out[f], k) for f in formulations for k in ("normal", "offset", "residual", "curvature",
                                                                     "status")]
    fmask = 0
    outs = (N.RfPixelOut * N.RF_NUM_FORMULATIONS)()
    for f in formulations:
        fmask |= 1 << _FORM_ID[f]
        outs[_FORM_ID[f]] = out[f]._c(B, H, W, d.device)
    cur = torch.cuda.current_stream(d.device)
    if stream is None:
        stream = cur
    elif stream != cur:
        # the conversions above ran on the current stream: order the launch after them, and keep
        # the caching allocator from handing their memory out before `stream` is done with it
        stream.wait_stream(cur)
        for t in temps:
            t.record_stream(stream)
    st = N.load().rf_fit_pixels(
        maps.handle, d.data_ptr(), dtype, B, H, W, d.stride(-2), mptr, int(window), fmask,
        outs, ctypes.c_void_p(stream.cuda_stream),
    )
    N.check(st, "fit_pixels")
    if squeeze:
        return {f: PixelFits(*(getattr(out[f], k)[0] for k in ("normal", "offset", "residual", "curvature", "status")))
                for f in formulations}
    return {f: out[f] for f in formulations}


class HostPipeline:
    """Host frames in, host outputs out: the reference-facing call with host buffers.

    Frames stream through the device in chunks of ``chunk_frames``: the H2D copy of chunk
    i+1, the fit kernels of chunk i and the D2H copies of chunk i-1 run concurrently on three
    streams (both PCIe directions and the SMs busy at once).  Device buffers are a ring of
    ``slots`` chunks, so device memory stays bounded for any batch; outputs land in pinned
    host ``PixelFits`` (allocated once per batch shape and reused).
    """

    def __init__(self, maps: TanAngleMaps, window: int, formulations=PIXEL_FORMULATIONS, chunk_frames: int = 8,
                 slots: int = 2):
        if chunk_frames < 1 or slots < 2:
            raise ValueError("chunk_frames must be >= 1 and slots >= 2")
        self.maps, self.window, self.chunk, self.slots = maps, int(window), int(chunk_frames), int(slots)
        self.formulations = (formulations,) if isinstance(formulations, str) else tuple(formulations)
        for f in self.formulations:
            if f not in _FORM_ID:
                raise ValueError(f"unknown formulation {f!r}; expected one of {FORMULATIONS}")
        self.device = torch.device("cuda", maps.device)
        self.h2d = torch.cuda.Stream(self.device)
        self.compute = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        self._dev_in = None
        self._dev_out = None
        self._host_out = None

    def _buffers(self, B: int, dtype: torch.dtype, host: bool = True):
        H, W, c = self.maps.height, self.maps.width, self.chunk
        if self._dev_in is None or self._dev_in.dtype != dtype:
            self._dev_in = torch.empty((self.slots, c, H, W), dtype=dtype, device=self.device)
            self._dev_out = [{f: PixelFits.empty(c, H, W, self.device) for f in self.formulations}
                             for _ in range(self.slots)]
        if host and (self._host_out is None or self._host_out[self.formulations[0]].status.shape[0] != B):
            pin = dict(pin_memory=True)
            self._host_out = {f: PixelFits(torch.empty((B, H, W, 3), **pin), torch.empty((B, H, W), **pin),
                                           torch.empty((B, H, W), **pin), torch.empty((B, H, W), **pin),
                                           torch.empty((B, H, W), dtype=torch.uint8, **pin))
                              for f in self.formulations}

    def run(self, depth: torch.Tensor, out: dict | None = None) -> dict:
        """depth: host tensor [B, H, W] (float32/float64 metres or uint16 mm; pinned for
        asynchronous copies).  Returns ``{formulation: PixelFits}`` of pinned host tensors,
        complete when this returns and reused by the next ``run`` of the same batch size;
        ``out`` (host PixelFits per formulation, [B, ...] each) receives them instead."""
        if depth.is_cuda:
            raise ValueError("HostPipeline.run takes host frames; use fit_pixels for device tensors")
        d = depth.unsqueeze(0) if depth.dim() == 2 else depth
        if d.dim() != 3 or tuple(d.shape[1:]) != (self.maps.height, self.maps.width):
            raise ValueError(f"depth must be [B, {self.maps.height}, {self.maps.width}], got {tuple(depth.shape)}")
        _depth_dtype(d)  # validates the element type
        d = d.contiguous()
        B = d.shape[0]
        self._buffers(B, d.dtype if out is None else d.dtype, host=out is None)
        host_out = self._host_out if out is None else out
        slot_free = [None] * self.slots   # D2H done with the slot's outputs (and the fit with its input)
        for i, b0 in enumerate(range(0, B, self.chunk)):
            b1 = min(B, b0 + self.chunk)
            k = i % self.slots
            src = self._dev_in[k, :b1 - b0]
            if slot_free[k] is not None:
                self.h2d.wait_event(slot_free[k])
            with torch.cuda.stream(self.h2d):
                src.copy_(d[b0:b1], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(self.h2d)
            self.compute.wait_event(ev_in)
            outs = {f: PixelFits(*(t[:b1 - b0] for t in (o.normal, o.offset, o.residual, o.curvature, o.status)))
                    for f, o in self._dev_out[k].items()}
            fit_pixels(src, self.maps, self.window, self.formulations, out=outs, stream=self.compute)
            ev_fit = torch.cuda.Event()
            ev_fit.record(self.compute)
            self.d2h.wait_event(ev_fit)
            with torch.cuda.stream(self.d2h):
                for f in self.formulations:
                    for name in ("normal", "offset", "residual", "curvature", "status"):
                        getattr(host_out[f], name)[b0:b1].copy_(getattr(outs[f], name), non_blocking=True)
                ev_out = torch.cuda.Event()
                ev_out.record(self.d2h)
            slot_free[k] = ev_out
        self.d2h.synchronize()
        return host_out


def launches_per_call(formulations=PIXEL_FORMULATIONS, window: int = 5, dtype=torch.float32,
                      shape: tuple = (64, 480, 640)) -> int:
    """Kernel launches one ``fit_pixels`` call over a ``shape`` = (B, H, W) batch issues
    (separable cameras, current device)."""
    fmask = 0
    for f in formulations:
        fmask |= 1 << _FORM_ID[f]
    code = {torch.float32: N.RF_DEPTH_F32_M, torch.float64: N.RF_DEPTH_F64_M}.get(dtype, N.RF_DEPTH_U16_MM)
    B, H, W = shape
    return int(N.load().rf_launches_per_call(fmask, int(window), code, int(B), int(H), int(W)))

"""B200-native per-pixel windowed plane fit (disparity-form and standard),
a drop-in for the fitting hot path of the reference package ``rangefit``
(arxiv/paper_2103_06644).  See DESIGN.md and include/rangefit_b200.h."""

from .pixels import (
    EXPLICIT_RGBD,
    EXPLICIT_STANDARD,
    FORMULATIONS,
    IMPLICIT_RGBD,
    IMPLICIT_STANDARD,
    MIN_SAMPLES,
    PIXEL_FORMULATIONS,
    STATUS_DEGENERATE,
    STATUS_FIT,
    STATUS_INPUT_VALID,
    CameraIntrinsics,
    PixelFits,
    TanAngleMaps,
    compute_tan_maps,
    fit_pixels,
    launches_per_call,
)

__all__ = [
    "EXPLICIT_RGBD",
    "EXPLICIT_STANDARD",
    "FORMULATIONS",
    "IMPLICIT_RGBD",
    "IMPLICIT_STANDARD",
    "MIN_SAMPLES",
    "PIXEL_FORMULATIONS",
    "STATUS_DEGENERATE",
    "STATUS_FIT",
    "STATUS_INPUT_VALID",
    "CameraIntrinsics",
    "PixelFits",
    "TanAngleMaps",
    "compute_tan_maps",
    "fit_pixels",
    "launches_per_call",
]

"""B200-native per-pixel windowed plane fit (disparity-form and standard),
a drop-in for the fitting hot path of the reference package ``rangefit``
(arxiv/paper_2103_06644).  See DESIGN.md and include/rangefit_b200.h."""

from .pixels import (
    IMPLICIT_RGBD,
    IMPLICIT_STANDARD,
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
    "IMPLICIT_RGBD",
    "IMPLICIT_STANDARD",
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

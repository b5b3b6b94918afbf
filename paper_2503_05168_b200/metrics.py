"""Image quality metrics on the GPU (drop-in for metrics.psnr / metrics.ssim,
pkg/src/seele/metrics.py:44-112): fp64 kernels in csrc/metrics.cu behind
``seele_psnr`` / ``seele_ssim``, so a rendered trajectory can be scored on the
device.  Inputs are (H, W, 3) arrays (numpy, or torch tensors on the device);
results are Python floats like the reference's."""
from __future__ import annotations

import numpy as np

from . import _native
from .errors import InvalidArgumentError

SSIM_WINDOW = 11


def _device_pair(img_a, img_b):
    import torch

    def dev(x):
        if isinstance(x, torch.Tensor):
            return x.to(device="cuda", dtype=torch.float64).contiguous()
        return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)), device="cuda")

    a, b = dev(img_a), dev(img_b)
    if tuple(a.shape) != tuple(b.shape):
        raise InvalidArgumentError(f"image shapes differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    return a, b


def psnr(img_a, img_b) -> float:
    """metrics.py:44-54: peak signal-to-noise ratio in dB for unit-range
    images; identical inputs give +inf."""
    import torch

    a, b = _device_pair(img_a, img_b)
    lib = _native.load()
    scratch = torch.empty(1024, dtype=torch.float64, device=a.device)
    out = torch.empty(1, dtype=torch.float64, device=a.device)
    _native.check(lib.seele_psnr(a.data_ptr(), b.data_ptr(), a.numel(), scratch.data_ptr(), out.data_ptr(),
                                 torch.cuda.current_stream(a.device).cuda_stream))
    return float(out.item())


def ssim(img_a, img_b) -> float:
    """metrics.py:72-112: mean structural similarity over the BT.601
    luminance, Gaussian 11x11 windows (sigma 1.5) where they fit."""
    import torch

    a, b = _device_pair(img_a, img_b)
    if a.dim() != 3 or a.shape[2] != 3:
        raise InvalidArgumentError("ssim expects (H, W, 3) images")
    h, w = int(a.shape[0]), int(a.shape[1])
    if min(h, w) < SSIM_WINDOW:
        raise InvalidArgumentError(f"images must be at least {SSIM_WINDOW} pixels per side for SSIM")
    lib = _native.load()
    scratch = torch.empty(int(lib.seele_metrics_scratch_doubles(w, h)), dtype=torch.float64, device=a.device)
    out = torch.empty(1, dtype=torch.float64, device=a.device)
    _native.check(lib.seele_ssim(a.data_ptr(), b.data_ptr(), w, h, scratch.data_ptr(), out.data_ptr(),
                                 torch.cuda.current_stream(a.device).cuda_stream))
    return float(out.item())

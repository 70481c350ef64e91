"""Residual bundle on the device (ref: residuals.py:193-296).

The sqrt-L1 / sqrt-(1-SSIM) residuals, grad_r_sq and color_grad are
computed by one fp64 kernel pair (csrc/residuals.cu); the float4 per-pixel
copies feed the product kernels, the (H, W, 3) float64 maps mirror the
reference's ResidualBundle fields.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .engine import LossConfig, ViewFrame, residual_pass
from .errors import ImageSizeError
from .scene import Camera


@dataclass
class ResidualBundle:
    mode: str
    lambda1: float
    lambda2: float
    r_abs: torch.Tensor
    r_ssim: torch.Tensor | None
    grad_r_sq: torch.Tensor
    color_grad: torch.Tensor
    drabs_dc: torch.Tensor
    drssim_dc: torch.Tensor | None
    energy: float
    gradr4: torch.Tensor   # (HW*4,) float32, product-kernel layout
    cgrad4: torch.Tensor

    @property
    def height(self) -> int:
        return self.r_abs.shape[0]

    @property
    def width(self) -> int:
        return self.r_abs.shape[1]

    @property
    def n_slots(self) -> int:
        return self.r_abs.numel()

    def residual_vector(self) -> torch.Tensor:
        if self.mode == "l2":
            return self.r_abs.reshape(-1).clone()
        return torch.cat([self.r_abs.reshape(-1), self.r_ssim.reshape(-1)])


def compute_residuals(rendered, gt, lambda1: float = 0.8, lambda2: float = 0.2, mode: str = "l1ssim",
                      window: int = 11, sigma: float = 1.5, eps_den: float = 1e-8) -> ResidualBundle:
    """ref: residuals.py:249-296."""
    rendered = torch.as_tensor(rendered)
    gt = torch.as_tensor(gt)
    if tuple(rendered.shape) != tuple(gt.shape):
        raise ImageSizeError(f"image shapes differ: {tuple(rendered.shape)} vs {tuple(gt.shape)}")
    if rendered.dim() != 3 or rendered.shape[2] != 3:
        raise ImageSizeError(f"expected (H, W, 3) images, got {tuple(rendered.shape)}")
    H, W = int(rendered.shape[0]), int(rendered.shape[1])
    dev = rendered.device
    fr = ViewFrame(Camera(torch.eye(3).numpy(), [0, 0, 0], 1.0, 1.0, 0.0, 0.0, W, H), 0)
    fr.rgb = rendered.to(torch.float64).contiguous().reshape(-1)
    loss = LossConfig(lambda1, lambda2, mode, window, sigma, eps_den)
    g4 = torch.zeros(H * W * 4, dtype=torch.float32, device=dev)
    c4 = torch.zeros(H * W * 4, dtype=torch.float32, device=dev)
    ex = {}
    part = residual_pass(fr, gt.to(dev), loss, g4, c4, ex)
    shp = (H, W, 3)
    l2 = mode == "l2"
    return ResidualBundle(mode=mode, lambda1=lambda1, lambda2=lambda2, r_abs=ex["rabs"].view(shp),
                          r_ssim=None if l2 else ex["rssim"].view(shp), grad_r_sq=ex["gradr"].view(shp),
                          color_grad=ex["cgrad"].view(shp), drabs_dc=ex["drabs"].view(shp),
                          drssim_dc=None if l2 else ex["drssim"].view(shp), energy=float(part.sum().item()),
                          gradr4=g4, cgrad4=c4)

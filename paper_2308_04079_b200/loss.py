"""Device L1 + D-SSIM loss (optimizer.loss, optimizer.py:141-163) via gs_l1_dssim_loss."""
from __future__ import annotations

import ctypes

import torch

from . import _lib

_ws_cache: dict = {}


def _workspace(width: int, height: int, device) -> torch.Tensor:
    key = (width, height, str(device), torch.cuda.current_stream(device).cuda_stream)
    ws = _ws_cache.get(key)
    if ws is None:
        nbytes = ctypes.c_size_t(0)
        _lib.check(_lib.load().gs_loss_workspace_size(width, height, ctypes.byref(nbytes)), "loss")
        ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws


def l1_dssim_loss(render: torch.Tensor, ground_truth: torch.Tensor, lambda_dssim: float = 0.2):
    """(loss, d_loss/d_render) like the reference: loss is a (4,) device tensor
    [total, mean L1, mean SSIM, mean squared error]; read it with float(loss[0]).  Raises
    ValueError on a resolution mismatch (optimizer.py:148-149)."""
    if tuple(render.shape) != tuple(ground_truth.shape):
        raise ValueError(f"resolution mismatch: {tuple(render.shape)} vs {tuple(ground_truth.shape)}")
    if render.dim() != 3 or render.shape[2] != 3:
        raise ValueError("images must be (H, W, 3)")
    if not 0.0 <= lambda_dssim <= 1.0:
        raise ValueError("lambda_dssim must be in [0, 1]")
    h, w = int(render.shape[0]), int(render.shape[1])
    render = render.detach().to(torch.float32).contiguous()
    ground_truth = ground_truth.detach().to(device=render.device, dtype=torch.float32).contiguous()
    ws = _workspace(w, h, render.device)
    loss = torch.empty(4, dtype=torch.float32, device=render.device)
    d_image = torch.empty_like(render)
    _lib.check(_lib.load().gs_l1_dssim_loss(render.data_ptr(), ground_truth.data_ptr(), w, h, float(lambda_dssim),
                                            ws.data_ptr(), ws.numel(), loss.data_ptr(), d_image.data_ptr(),
                                            torch.cuda.current_stream(render.device).cuda_stream), "loss")
    return loss, d_image

"""Batched mapping across GPUs: the host-side plumbing around the C ABI.

Mapping a section renders several keyframe views of it and minimises the sum of their
Eq. 2 losses (§3.4) over the section's learnable Gaussians.  The views are
independent given the Gaussian state, so they shard across ranks with ONE exchange per step:
every rank holds the same section (each instantiates it locally — deterministic, no
broadcast), renders its slice of the views with `vtgs_render_fwd`, accumulates the attribute
gradients of all of them into one contiguous 5N fp32 buffer with `vtgs_render_bwd` (+=), and a
single sum all-reduce (NCCL over NVLink 5 / NVSwitch on the GPU box, gloo in the CPU tests)
makes the buffer identical on every rank.  Tracking a single view does not shard (replicas
only); its pose gradient is reduced on the device.

This module is argument marshalling and collective plumbing only; every step of the method runs
in libvtgs.so.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch
import torch.distributed as dist


def shard_views(n_views: int, world_size: int, rank: int) -> List[int]:
    """Contiguous, balanced view slice of `rank` (sizes differ by at most one; every view is
    owned by exactly one rank; ranks beyond n_views get none)."""
    if world_size <= 0 or not 0 <= rank < world_size:
        raise ValueError("bad world_size / rank")
    base, extra = divmod(n_views, world_size)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


class GradBuffer:
    """One contiguous fp32 buffer holding d_col_opa (N×4) followed by d_radius (N) — the layout
    that lets a single all-reduce move every attribute gradient of the section."""

    def __init__(self, n: int, device):
        self.n = n
        self.flat = torch.zeros(5 * n, dtype=torch.float32, device=device)
        self.d_col_opa = self.flat[: 4 * n].view(n, 4)
        self.d_radius = self.flat[4 * n:]

    def zero_(self):
        self.flat.zero_()
        return self


def allreduce_grads(buf: GradBuffer, group: Optional[dist.ProcessGroup] = None) -> GradBuffer:
    """Sum the gradient buffer over the ranks of `group` (no-op without a process group)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf.flat, op=dist.ReduceOp.SUM, group=group)
    return buf


class BatchedMapper:
    """Per-rank driver of one mapping step over a shard of views: the fused masked-L1 terms of
    Eq. 2, plus its SSIM term τ·L_S when `w_ssim` = τ > 0 (τ = 0.2 at P:262)."""

    def __init__(self, renderer, pos_rad: torch.Tensor, col_opa: torch.Tensor, intr,
                 views: Sequence[torch.Tensor], targets: Sequence[dict], w_color: float, w_depth: float,
                 learn: Sequence[int] = (0, 1 << 62), group: Optional[dist.ProcessGroup] = None,
                 w_ssim: float = 0.0):
        from . import vtgs
        self.vt = vtgs
        self.R = renderer
        self.pos_rad, self.col_opa, self.intr = pos_rad, col_opa, intr
        self.views = list(views)
        self.targets = list(targets)
        self.w_color, self.w_depth = float(w_color), float(w_depth)
        self.learn = learn
        self.group = group
        n = pos_rad.shape[0]
        self.grads = GradBuffer(n, pos_rad.device)
        H, W = intr.height, intr.width
        dev = pos_rad.device
        self.out = (torch.empty((H, W, 3), device=dev), torch.empty((H, W), device=dev),
                    torch.empty((H, W), device=dev))
        self.loss = torch.zeros(max(len(self.views), 1), device=dev)
        self.w_ssim = float(w_ssim)
        self.ssim_loss = torch.zeros(max(len(self.views), 1), device=dev)
        self.d_ssim = torch.zeros((H, W, 3), device=dev) if self.w_ssim > 0 else None

    def step(self, allreduce: bool = True, check: Optional[bool] = None) -> GradBuffer:
        """Zero the gradients, render + backprop every local view (accumulating), all-reduce.
        `check` (default: on the first step) synchronises once and raises VtgsError if a view's
        tile pairs exceeded the context's capacity (the render would silently be empty)."""
        if check is None:
            check = not getattr(self, "_checked", False)
        self.grads.zero_()
        for i, (v, t) in enumerate(zip(self.views, self.targets)):
            self.R.render_fwd(self.pos_rad, self.col_opa, v, self.intr, out=self.out)
            if self.d_ssim is not None:
                self.d_ssim.zero_()
                self.R.ssim_loss(self.out[0], t["rgb"], self.w_ssim, d_color=self.d_ssim,
                                 loss_out=self.ssim_loss[i:i + 1])
            self.R.render_bwd(self.vt.VTGS_GRAD_ATTR, d_col_opa=self.grads.d_col_opa, d_radius=self.grads.d_radius,
                              loss=dict(target_rgb=t["rgb"], target_depth=t["depth"], w_color=self.w_color,
                                        w_depth=self.w_depth, extra_dcolor=self.d_ssim),
                              learn=self.learn, loss_out=self.loss[i:i + 1])
        if check:
            self.R.check()
            self._checked = True
        if allreduce:
            allreduce_grads(self.grads, self.group)
        return self.grads

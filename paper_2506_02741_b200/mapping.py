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
    Eq. 2, plus its SSIM term τ·L_S when `w_ssim` = τ > 0 (τ = 0.2 at P:262).

    `renderer` may be a list of renderer contexts: view i then renders on context i mod k, each on
    its own CUDA stream forked from (and joined back into) the caller's, so consecutive views'
    kernels overlap on the GPU (one view's tail waves under the next view's first ones).  The
    views write the shared gradient buffer with float atomics only (commutative), so the result is
    the same sum; the deterministic merge finalises per context and is not combined with k > 1."""

    def __init__(self, renderer, pos_rad: torch.Tensor, col_opa: torch.Tensor, intr,
                 views: Sequence[torch.Tensor], targets: Sequence[dict], w_color: float, w_depth: float,
                 learn: Sequence[int] = (0, 1 << 62), group: Optional[dist.ProcessGroup] = None,
                 w_ssim: float = 0.0, deterministic: bool = False):
        from . import vtgs
        self.vt = vtgs
        self.Rs = list(renderer) if isinstance(renderer, (list, tuple)) else [renderer]
        self.R = self.Rs[0]
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
        k = len(self.Rs)
        self.outs = [(torch.empty((H, W, 3), device=dev), torch.empty((H, W), device=dev),
                      torch.empty((H, W), device=dev)) for _ in range(k)]
        self.out = self.outs[0]
        self.loss = torch.zeros(max(len(self.views), 1), device=dev)
        self.w_ssim = float(w_ssim)
        self.ssim_loss = torch.zeros(max(len(self.views), 1), device=dev)
        self.d_ssims = [torch.zeros((H, W, 3), device=dev) if self.w_ssim > 0 else None for _ in range(k)]
        self.d_ssim = self.d_ssims[0]
        self.streams = [torch.cuda.Stream(dev) for _ in range(k)] if k > 1 else None
        if deterministic and k > 1:
            raise ValueError("the deterministic merge finalises per context: use one renderer context")
        # VTGS_GRAD_DETERMINISTIC: int64 fixed-point merge of the attribute gradients
        self.want = vtgs.VTGS_GRAD_ATTR | (vtgs.VTGS_GRAD_DETERMINISTIC if deterministic else 0)

    def _view(self, i, v, t):
        j = i % len(self.Rs)
        R, out, d_ssim = self.Rs[j], self.outs[j], self.d_ssims[j]
        R.render_fwd(self.pos_rad, self.col_opa, v, self.intr, out=out)
        if d_ssim is not None:
            d_ssim.zero_()
            R.ssim_loss(out[0], t["rgb"], self.w_ssim, d_color=d_ssim, loss_out=self.ssim_loss[i:i + 1])
        R.render_bwd(self.want, d_col_opa=self.grads.d_col_opa, d_radius=self.grads.d_radius,
                     loss=dict(target_rgb=t["rgb"], target_depth=t["depth"], w_color=self.w_color,
                               w_depth=self.w_depth, extra_dcolor=d_ssim),
                     learn=self.learn, loss_out=self.loss[i:i + 1])

    def step(self, allreduce: bool = True, check: Optional[bool] = None, serial: bool = False) -> GradBuffer:
        """Zero the gradients, render + backprop every local view (accumulating), all-reduce.
        `check` (default: on the first step) synchronises once and raises VtgsError if a view's
        tile pairs exceeded the context's capacity (the render would silently be empty).
        `serial` runs the views one after another on the caller's stream even with several
        contexts (per-kernel event timing is only meaningful without concurrent kernels)."""
        if check is None:
            check = not getattr(self, "_checked", False)
        self.grads.zero_()
        if self.streams is None or serial:
            for i, (v, t) in enumerate(zip(self.views, self.targets)):
                self._view(i, v, t)
        else:   # fork: every context's stream starts after the zeroing; join before the all-reduce
            cur = torch.cuda.current_stream(self.pos_rad.device)
            for s in self.streams:
                s.wait_stream(cur)
            for i, (v, t) in enumerate(zip(self.views, self.targets)):
                with torch.cuda.stream(self.streams[i % len(self.streams)]):
                    self._view(i, v, t)
            for s in self.streams:
                cur.wait_stream(s)
        if check:
            for j, R in enumerate(self.Rs):
                R.check(stream=self.streams[j] if self.streams and not serial else None)
            self._checked = True
        if allreduce:
            allreduce_grads(self.grads, self.group)
        return self.grads

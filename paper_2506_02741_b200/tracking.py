"""Tracking drivers (host orchestration around the C ABI; every step runs in libvtgs.so).

* `track(...)` — one frame: `iterations` × (render_fwd → fused masked-L1 of Eq. 1 with the
  tracking mask W_i → pose backward → device Adam), PAPER.md:137-146 (§3.3, Eq. 1), optionally
  captured in one CUDA graph (launch-only loop: the view pose is a device buffer).
* `pretrack_select(...)` — the head-frame pre-tracking of PAPER.md:180-182 (§3.3, "Selecting
  Overlapping Section S^o": "We use each one of the 3 sections to conduct the tracking for
  several iterations, respectively. We eventually select a section that produces the minimum
  rendering error as S^o").  The candidates are independent (each owns its pose copy and
  reads its frozen section), so each runs on its own renderer context and CUDA stream,
  concurrently on one GPU (or one per GPU); the selection is the argmin of the final losses.
* `section_visibility(...)` — W_i's visibility term: the union of the frame's visibility to the
  section's head, middle and last frames (vtgs_visibility_mask).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import torch


@dataclass
class TrackResult:
    pose: torch.Tensor            # [1, 7] device
    losses: torch.Tensor          # [iterations] device, the Eq. 1 loss at each iterate
    final_loss: float = field(default=float("nan"))


def section_visibility(renderer, depth: torch.Tensor, pose: torch.Tensor, kf_depth: torch.Tensor,
                       kf_poses: torch.Tensor, intr, tol: float = 0.01) -> torch.Tensor:
    """Visibility mask of a frame to a section: union over the section's head, middle and last
    keyframes (middle = ⌊K/2⌋)."""
    K = kf_depth.shape[0]
    idx = sorted({0, K // 2, K - 1})
    return renderer.visibility_mask(depth, pose, kf_depth[idx].contiguous(), kf_poses[idx].contiguous(), intr, tol)


def track(renderer, pos_rad: torch.Tensor, col_opa: torch.Tensor, intr, rgb: torch.Tensor, depth: torch.Tensor,
          init_pose: torch.Tensor, iterations: int, lr_rot: float, lr_trans: float, w_color: float = 0.5,
          w_depth: float = 1.0, vis_mask: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None,
          graph: bool = False) -> TrackResult:
    """Optimise the frame's 7 pose parameters against the frozen Gaussians (Eq. 1, mean form,
    W_i = valid ∧ S > 0.99 ∧ vis).  Returns the final pose and the per-iteration losses."""
    from . import vtgs
    dev = pos_rad.device
    H, W = intr.height, intr.width
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.stream(s):   # the loop's buffers are initialised on its own stream
        pose = init_pose.reshape(1, 7).clone()
        state = torch.zeros(16, device=dev)
        dp = torch.zeros(7, device=dev)
        losses = torch.zeros(iterations, device=dev)
        out = (torch.empty((H, W, 3), device=dev), torch.empty((H, W), device=dev), torch.empty((H, W), device=dev))
    L = dict(target_rgb=rgb, target_depth=depth, vis_mask=vis_mask, w_color=w_color, w_depth=w_depth,
             color_mask_mode=1, depth_mask_mode=1, normalize=1)

    def body():
        for i in range(iterations):
            renderer.render_fwd(pos_rad, col_opa, pose, intr, out=out, stream=s)
            renderer.render_bwd(vtgs.VTGS_GRAD_POSE, d_pose=dp, loss=L, loss_out=losses[i:i + 1], stream=s)
            renderer.pose_adam_step(pose, dp, state, lr_rot, lr_trans, stream=s)

    if graph:
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                body()
            pose.copy_(init_pose.reshape(1, 7))
            state.zero_()
            g.replay()
    else:
        with torch.cuda.stream(s):
            body()
    return TrackResult(pose, losses)


def pretrack_select(renderers: Sequence, sections: Sequence[dict], intr, rgb: torch.Tensor, depth: torch.Tensor,
                    init_pose: torch.Tensor, iterations: int, lr_rot: float, lr_trans: float,
                    w_color: float = 0.5, w_depth: float = 1.0, concurrent: bool = True):
    """Pre-track the head frame against each candidate section (dict(pos_rad, col_opa[, vis_mask]))
    for `iterations` and select the one with the minimum final rendering error.
    One renderer context per candidate (contexts own their scratch); with `concurrent` each runs
    on its own CUDA stream.  Returns (best index, [final losses], [TrackResult])."""
    assert len(renderers) == len(sections)
    dev = rgb.device
    streams = [torch.cuda.Stream(dev) for _ in sections] if concurrent else [torch.cuda.current_stream(dev)] * len(sections)
    cur = torch.cuda.current_stream(dev)
    results: List[TrackResult] = []
    for R, sec, s in zip(renderers, sections, streams):
        s.wait_stream(cur)
        results.append(track(R, sec["pos_rad"], sec["col_opa"], intr, rgb, depth, init_pose, iterations, lr_rot,
                             lr_trans, w_color, w_depth, sec.get("vis_mask"), stream=s))
    for s in streams:
        cur.wait_stream(s)
    torch.cuda.synchronize(dev)
    finals = [float(r.losses[-1].item()) for r in results]
    for r, f in zip(results, finals):
        r.final_loss = f
    best = min(range(len(finals)), key=lambda i: finals[i])
    return best, finals, results

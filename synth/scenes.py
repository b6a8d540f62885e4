"""Seeded synthetic RGB-D inputs shaped like the paper's workloads.

This module is the ONE place that both the CUDA path (tests, bench) and the CPU oracle
(tests only) take their inputs from.  It holds none of the method's arithmetic: no
back-projection into Gaussians, no projection, no splatting.  It only ray-casts procedural
box scenes into depth/RGB images along a trajectory of camera poses, the way an RGB-D sensor
would observe them, and draws the per-Gaussian opacities the configs prescribe.

Why synthetic: the paper evaluates on Replica / TUM-RGBD / ScanNet / ScanNet++ / KITTI
(§4 "Dataset and Metrics", Supp.).  None of them is in this
container, so these seeded scenes stand in for them, with the shapes, intrinsics and depth
ranges that BASELINE.json's five configs state (see DESIGN.md §"Input recipe").

Conventions (SPEC.md:29-34 `Pose`; SURVEY.md §8(c) readings 10-11):
  * pose = camera-to-world, unit quaternion (w, x, y, z) + translation (metres);
  * OpenCV camera axes: x right, y down, z forward; pixel (x, y) has its centre at integer
    coordinates (x, y); depth is z-depth in metres, 0 = invalid.
All randomness comes from numpy PCG64 generators seeded per component.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "Intrinsics", "Frame", "Scene", "rotmat_to_quat", "quat_to_rotmat", "pose_compose",
    "perturb_pose", "make_config", "CONFIG_NAMES",
]


# ----------------------------------------------------------------------------------------
# small pose helpers (fp64, input generation only)
# ----------------------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Intrinsics:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int


def quat_to_rotmat(q: Sequence[float]) -> np.ndarray:
    w, x, y, z = (float(v) for v in q)
    n = math.sqrt(w * w + x * x + y * y + z * z)
    w, x, y, z = w / n, x / n, y / n, z / n
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def rotmat_to_quat(R: np.ndarray) -> np.ndarray:
    """Shepperd's method; returns (w, x, y, z) with w >= 0."""
    R = np.asarray(R, dtype=np.float64)
    tr = R[0, 0] + R[1, 1] + R[2, 2]
    if tr > 0:
        s = math.sqrt(tr + 1.0) * 2
        q = [0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s]
    elif R[0, 0] > R[1, 1] and R[0, 0] > R[2, 2]:
        s = math.sqrt(1.0 + R[0, 0] - R[1, 1] - R[2, 2]) * 2
        q = [(R[2, 1] - R[1, 2]) / s, 0.25 * s, (R[0, 1] + R[1, 0]) / s, (R[0, 2] + R[2, 0]) / s]
    elif R[1, 1] > R[2, 2]:
        s = math.sqrt(1.0 + R[1, 1] - R[0, 0] - R[2, 2]) * 2
        q = [(R[0, 2] - R[2, 0]) / s, (R[0, 1] + R[1, 0]) / s, 0.25 * s, (R[1, 2] + R[2, 1]) / s]
    else:
        s = math.sqrt(1.0 + R[2, 2] - R[0, 0] - R[1, 1]) * 2
        q = [(R[1, 0] - R[0, 1]) / s, (R[0, 2] + R[2, 0]) / s, (R[1, 2] + R[2, 1]) / s, 0.25 * s]
    q = np.array(q)
    q /= np.linalg.norm(q)
    if q[0] < 0:
        q = -q
    return q


def axis_angle_to_rotmat(axis: np.ndarray, angle: float) -> np.ndarray:
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(angle) * K + (1 - math.cos(angle)) * (K @ K)


def pose_to_Rt(pose: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    pose = np.asarray(pose, dtype=np.float64)
    return quat_to_rotmat(pose[:4]), pose[4:7].copy()


def Rt_to_pose(R: np.ndarray, t: np.ndarray) -> np.ndarray:
    return np.concatenate([rotmat_to_quat(R), np.asarray(t, dtype=np.float64)])


def pose_compose(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """a ∘ b for camera-to-world poses (apply b first, then a)."""
    Ra, ta = pose_to_Rt(a)
    Rb, tb = pose_to_Rt(b)
    return Rt_to_pose(Ra @ Rb, Ra @ tb + ta)


def perturb_pose(pose: np.ndarray, rot_deg: float, trans_m: float, rng: np.random.Generator) -> np.ndarray:
    """pose ∘ δ, δ = rotation of `rot_deg` about a uniform random axis and a translation of
    length `trans_m` in a uniform random direction (SURVEY.md §8(d) config 1/3 recipe)."""
    axis = rng.normal(size=3)
    direction = rng.normal(size=3)
    direction /= np.linalg.norm(direction)
    delta = Rt_to_pose(axis_angle_to_rotmat(axis, math.radians(rot_deg)), trans_m * direction)
    return pose_compose(pose, delta)


def look_pose(position: np.ndarray, yaw: float, pitch: float) -> np.ndarray:
    """Camera-to-world pose of an OpenCV camera at `position` looking along heading (yaw, pitch)
    in a z-up world."""
    f = np.array([math.cos(yaw) * math.cos(pitch), math.sin(yaw) * math.cos(pitch), math.sin(pitch)])
    right = np.cross(f, [0.0, 0.0, 1.0])
    right /= np.linalg.norm(right)
    down = np.cross(f, right)
    R = np.stack([right, down, f], axis=1)
    return Rt_to_pose(R, position)


# ----------------------------------------------------------------------------------------
# procedural box scenes + ray casting
# ----------------------------------------------------------------------------------------
@dataclasses.dataclass
class Box:
    lo: np.ndarray
    hi: np.ndarray
    base: np.ndarray          # (6, 3) base colour per face
    grad: np.ndarray          # (6, 2, 3) linear colour gradient per face along its 2 in-plane axes


@dataclasses.dataclass
class Scene:
    shell_lo: np.ndarray      # the room shell (rays exit it)
    shell_hi: np.ndarray
    shell: Box
    solids: List[Box]         # axis-aligned solids (furniture boxes, interior walls)


def _face_colours(rng: np.random.Generator) -> Tuple[np.ndarray, np.ndarray]:
    base = rng.uniform(0.15, 0.85, size=(6, 3))
    grad = rng.uniform(-0.25, 0.25, size=(6, 2, 3))
    return base, grad


def _make_box(lo, hi, rng) -> Box:
    base, grad = _face_colours(rng)
    return Box(np.asarray(lo, dtype=np.float64), np.asarray(hi, dtype=np.float64), base, grad)


def _room_scene(size: Sequence[float], n_boxes: int, rng: np.random.Generator,
                walls: Sequence[Tuple[Sequence[float], Sequence[float]]] = (),
                keepout: Sequence[Tuple[float, float, float]] = ()) -> Scene:
    """Room [0,size] (z-up) with `n_boxes` random axis-aligned boxes standing on the floor,
    sizes U(0.3, 1.2) m, plus optional interior wall slabs. `keepout` is a
    list of (x, y, radius) discs no box may intrude on (keeps the camera path clear)."""
    size = np.asarray(size, dtype=np.float64)
    shell = _make_box([0.0, 0.0, 0.0], size, rng)
    solids: List[Box] = []
    for lo, hi in walls:
        solids.append(_make_box(lo, hi, rng))
    tries = 0
    while len(solids) < len(walls) + n_boxes and tries < 10000:
        tries += 1
        ext = rng.uniform(0.3, 1.2, size=3)
        ext[2] = min(ext[2], size[2] - 0.2)
        cx = rng.uniform(0.1 + ext[0] / 2, size[0] - 0.1 - ext[0] / 2)
        cy = rng.uniform(0.1 + ext[1] / 2, size[1] - 0.1 - ext[1] / 2)
        lo = np.array([cx - ext[0] / 2, cy - ext[1] / 2, 0.0])
        hi = np.array([cx + ext[0] / 2, cy + ext[1] / 2, ext[2]])
        ok = True
        for (kx, ky, kr) in keepout:
            dx = max(lo[0] - kx, 0.0, kx - hi[0])
            dy = max(lo[1] - ky, 0.0, ky - hi[1])
            if dx * dx + dy * dy < kr * kr:
                ok = False
                break
        if ok:
            for (wlo, whi) in walls:
                if (lo[0] < whi[0] + 0.05 and hi[0] > wlo[0] - 0.05 and lo[1] < whi[1] + 0.05
                        and hi[1] > wlo[1] - 0.05):
                    ok = False
                    break
        if ok:
            solids.append(_make_box(lo, hi, rng))
    return Scene(np.zeros(3), size, shell, solids)


def _clearance(scene: Scene, p: np.ndarray) -> float:
    """Distance from point p to the nearest shell wall / solid (inf-norm free, Euclidean)."""
    d = float(np.min(np.concatenate([p - scene.shell_lo, scene.shell_hi - p])))
    for b in scene.solids:
        q = np.maximum(np.maximum(b.lo - p, 0.0), p - b.hi)
        d = min(d, float(np.linalg.norm(q)))
    return d


def _face_uv(face: np.ndarray, pts: np.ndarray, lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """In-plane normalised coordinates (2 per point) of the face a point lies on."""
    axis = face // 2                       # 0,1: x faces; 2,3: y faces; 4,5: z faces
    ext = np.maximum(hi - lo, 1e-6)
    rel = (pts - lo) / ext
    uv = np.empty((pts.shape[0], 2))
    a0 = np.where(axis == 0, 1, 0)
    a1 = np.where(axis == 2, 1, 2)
    uv[:, 0] = np.take_along_axis(rel, a0[:, None], 1)[:, 0]
    uv[:, 1] = np.take_along_axis(rel, a1[:, None], 1)[:, 0]
    return uv


def ray_cast(scene: Scene, pose: np.ndarray, intr: Intrinsics, rng: np.random.Generator,
             invalid_frac: float = 0.01, depth_range=(0.3, 6.0)) -> Tuple[np.ndarray, np.ndarray]:
    """Render z-depth (m, 0 = invalid) and RGB in [0,1] of `scene` from camera-to-world `pose`.
    Depth invalid if no hit, outside `depth_range`, or Bernoulli(`invalid_frac`)."""
    W, H = intr.width, intr.height
    R, t = pose_to_Rt(pose)
    xs = (np.arange(W, dtype=np.float64) - intr.cx) / intr.fx
    ys = (np.arange(H, dtype=np.float64) - intr.cy) / intr.fy
    dc = np.stack(np.broadcast_arrays(xs[None, :], ys[:, None], np.ones((H, W))), axis=-1).reshape(-1, 3)
    dw = dc @ R.T                                  # ray directions with unit camera-z
    n = dw.shape[0]
    inv = 1.0 / np.where(np.abs(dw) < 1e-12, 1e-12, dw)
    best_t = np.full(n, np.inf)
    best_obj = np.full(n, -1, dtype=np.int64)      # -1 shell, k solid k
    best_face = np.zeros(n, dtype=np.int64)
    # shell: exit distance (ray starts inside)
    t1 = (scene.shell_lo - t) * inv
    t2 = (scene.shell_hi - t) * inv
    tmax_axis = np.maximum(t1, t2)
    exit_axis = np.argmin(tmax_axis, axis=1)
    t_exit = tmax_axis[np.arange(n), exit_axis]
    hit_hi = np.take_along_axis(t2 >= t1, exit_axis[:, None], 1)[:, 0]
    best_t = t_exit
    best_face = exit_axis * 2 + hit_hi.astype(np.int64)
    all_idx = np.arange(n)
    for k, b in enumerate(scene.solids):
        # rays that can hit the box: its 8 corners' image bbox (+2 px) when all are in front of
        # the camera, else every ray (a speed-up only; the per-ray arithmetic is unchanged)
        corners = np.array([[x, y, z] for x in (b.lo[0], b.hi[0]) for y in (b.lo[1], b.hi[1])
                            for z in (b.lo[2], b.hi[2])])
        cc = (corners - t) @ R
        if np.all(cc[:, 2] > 0.05):
            uu = intr.fx * cc[:, 0] / cc[:, 2] + intr.cx
            vv = intr.fy * cc[:, 1] / cc[:, 2] + intr.cy
            x0, x1 = int(max(0, np.floor(uu.min()) - 2)), int(min(W - 1, np.ceil(uu.max()) + 2))
            y0, y1 = int(max(0, np.floor(vv.min()) - 2)), int(min(H - 1, np.ceil(vv.max()) + 2))
            if x0 > x1 or y0 > y1:
                continue
            idx = (np.arange(y0, y1 + 1)[:, None] * W + np.arange(x0, x1 + 1)[None, :]).reshape(-1)
        else:
            idx = all_idx
        t1 = (b.lo - t) * inv[idx]
        t2 = (b.hi - t) * inv[idx]
        tmin_axis = np.minimum(t1, t2)
        tmax_axis = np.maximum(t1, t2)
        ent_axis = np.argmax(tmin_axis, axis=1)
        t_ent = tmin_axis[np.arange(len(idx)), ent_axis]
        t_ex = np.min(tmax_axis, axis=1)
        hit = (t_ent <= t_ex) & (t_ent > 1e-6) & (t_ent < best_t[idx])
        if np.any(hit):
            hi_ = idx[hit]
            best_t[hi_] = t_ent[hit]
            best_obj[hi_] = k
            # entering through the low face of an axis when the ray moves +axis
            lo_face = np.take_along_axis(t1 <= t2, ent_axis[:, None], 1)[:, 0]
            best_face[hi_] = (ent_axis * 2 + (~lo_face).astype(np.int64))[hit]
    pts = t[None, :] + best_t[:, None] * dw
    rgb = np.empty((n, 3))
    objs = [scene.shell] + scene.solids
    for k in range(-1, len(scene.solids)):
        sel = np.nonzero(best_obj == k)[0]
        if sel.size == 0:
            continue
        b = objs[k + 1]
        f = best_face[sel]
        uv = _face_uv(f, pts[sel], b.lo, b.hi)
        col = b.base[f] + uv[:, 0:1] * b.grad[f, 0] + uv[:, 1:2] * b.grad[f, 1]
        rgb[sel] = col
    rgb += rng.uniform(0.0, 0.05, size=rgb.shape)
    rgb = np.clip(rgb, 0.0, 1.0)
    depth = best_t.copy()                          # z-depth because camera-z of dw is 1
    bad = (~np.isfinite(depth)) | (depth < depth_range[0]) | (depth > depth_range[1])
    bad |= rng.random(n) < invalid_frac
    depth[bad] = 0.0
    return depth.reshape(H, W).astype(np.float32), rgb.reshape(H, W, 3).astype(np.float32)


def _trajectory(scene: Scene, n: int, rng: np.random.Generator, step_m=0.10, step_deg=5.0,
                clearance=0.5, height=(1.2, 1.8), start=None) -> List[np.ndarray]:
    """Smooth random trajectory: every step translates exactly `step_m` and yaws exactly
    `step_deg` (pitch fixed), keeping `clearance` from every surface."""
    for _attempt in range(200):
        if start is None:
            p = np.array([rng.uniform(scene.shell_lo[0] + 0.7, scene.shell_hi[0] - 0.7),
                          rng.uniform(scene.shell_lo[1] + 0.7, scene.shell_hi[1] - 0.7),
                          rng.uniform(*height)])
        else:
            p = np.asarray(start, dtype=np.float64).copy()
        if _clearance(scene, p) < clearance:
            continue
        centre = 0.5 * (scene.shell_lo + scene.shell_hi)
        yaw = math.atan2(centre[1] - p[1], centre[0] - p[0]) + math.pi + rng.uniform(-0.5, 0.5)
        if np.linalg.norm(centre[:2] - p[:2]) > 0.5:
            yaw -= math.pi  # look across the room, towards (and past) its centre
        pitch = math.radians(rng.uniform(-15, 5))
        turn = 1.0 if rng.random() < 0.5 else -1.0
        poses = [look_pose(p, yaw, pitch)]
        ok = True
        for _ in range(n - 1):
            placed = False
            for _try in range(64):
                heading = yaw + rng.uniform(-math.pi / 2, math.pi / 2) if _try else yaw
                q = p + step_m * np.array([math.cos(heading), math.sin(heading), 0.0])
                if _clearance(scene, q) >= clearance:
                    placed = True
                    break
            if not placed:
                ok = False
                break
            if rng.random() < 0.15:
                turn = -turn
            yaw += turn * math.radians(step_deg)
            p = q
            poses.append(look_pose(p, yaw, pitch))
        if ok:
            return poses
    raise RuntimeError("could not place a trajectory with the requested clearance")


# ----------------------------------------------------------------------------------------
# the five BASELINE.json configs
# ----------------------------------------------------------------------------------------
@dataclasses.dataclass
class Frame:
    depth: np.ndarray          # f32 [H, W] metres, 0 = invalid
    rgb: np.ndarray            # f32 [H, W, 3] in [0, 1]
    pose: np.ndarray           # f64 [7] camera-to-world (w, x, y, z, tx, ty, tz)


@dataclasses.dataclass
class Config:
    name: str
    intr: Intrinsics
    keyframes: List[Frame]     # the section: every valid pixel of every keyframe ties a Gaussian
    opacity: np.ndarray        # f32 [K, H, W] = sigmoid(N(0,1)) initial opacities
    views: List[np.ndarray]    # render poses (f64 [7]) for this config's step
    targets: List[Frame]       # observation per view (loss targets)
    loss_weights: Tuple[float, float]
    mode: str                  # "mapping" | "tracking" | "full"
    seed: int
    extra: dict = dataclasses.field(default_factory=dict)

    @property
    def K(self) -> int:
        return len(self.keyframes)

    @property
    def n_slots(self) -> int:
        return self.K * self.intr.width * self.intr.height

    def depth_stack(self) -> np.ndarray:
        return np.stack([f.depth for f in self.keyframes])

    def rgb_stack(self) -> np.ndarray:
        return np.stack([f.rgb for f in self.keyframes])

    def pose_stack(self) -> np.ndarray:
        return np.stack([f.pose for f in self.keyframes]).astype(np.float32)


CONFIG_NAMES = {1: "tiny", 2: "mapping", 3: "tracking", 4: "batched_mapping", 5: "large"}


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def _config1(seed: int) -> Config:
    """64×48, fx=fy=60, cx=32, cy=24; one identity keyframe; depth = tilted plane whose 1/z is
    linear in x from 1/1.5 to 1/3.0 plus N(0, 0.01) m; RGB U[0,1]^3; o = sigmoid(N(0,1));
    render pose = keyframe ∘ (2°, 3 cm) (BASELINE.json configs[0])."""
    rng = np.random.Generator(np.random.PCG64(seed))
    intr = Intrinsics(60.0, 60.0, 32.0, 24.0, 64, 48)
    W, H = intr.width, intr.height
    inv = np.linspace(1 / 1.5, 1 / 3.0, W)[None, :].repeat(H, 0)
    depth = (1.0 / inv + rng.normal(0.0, 0.01, size=(H, W))).astype(np.float32)
    rgb = rng.uniform(0.0, 1.0, size=(H, W, 3)).astype(np.float32)
    kf = Frame(depth, rgb, np.array([1.0, 0, 0, 0, 0, 0, 0]))
    opacity = _sigmoid(rng.normal(size=(1, H, W))).astype(np.float32)
    view = perturb_pose(kf.pose, 2.0, 0.03, rng)
    return Config("tiny", intr, [kf], opacity, [view], [kf], (1.0, 0.5), "full", seed)


def _config_room(name: str, seed: int, intr: Intrinsics, size, n_boxes: int, n_kf: int) -> Tuple[Scene, List[np.ndarray], List[Frame], np.ndarray, np.random.Generator]:
    rng_scene = np.random.Generator(np.random.PCG64([seed, 1]))
    rng_traj = np.random.Generator(np.random.PCG64([seed, 2]))
    rng_img = np.random.Generator(np.random.PCG64([seed, 3]))
    rng_opa = np.random.Generator(np.random.PCG64([seed, 4]))
    scene = None
    for _ in range(50):
        scene = _room_scene(size, n_boxes, rng_scene)
        try:
            poses = _trajectory(scene, n_kf, rng_traj)
            break
        except RuntimeError:
            continue
    kfs = []
    for p in poses:
        d, c = ray_cast(scene, p, intr, rng_img)
        kfs.append(Frame(d, c, p))
    opacity = _sigmoid(rng_opa.normal(size=(n_kf, intr.height, intr.width))).astype(np.float32)
    return scene, poses, kfs, opacity, rng_img


def _config2(seed: int) -> Config:
    """Mapping: 5 keyframes 1200×680 (f=600, c=(599.5, 339.5)), room 6×5×3 m with 12 boxes;
    render keyframe 2's view against its RGB-D; loss 0.8·L1(C) + 1.0·U·L1(D)
    (ρ, σ of PAPER.md:262 §4; BASELINE.json configs[1])."""
    intr = Intrinsics(600.0, 600.0, 599.5, 339.5, 1200, 680)
    scene, poses, kfs, opacity, _ = _config_room("mapping", seed, intr, (6.0, 5.0, 3.0), 12, 5)
    return Config("mapping", intr, kfs, opacity, [kfs[2].pose], [kfs[2]], (0.8, 1.0), "mapping", seed)


def _config3(seed: int) -> Config:
    """Tracking: 10 keyframes 640×480 (f=525, c=(319.5, 239.5)); frame to track = half a step
    after keyframe 9, ray-cast at ground truth; init = GT ∘ (1.5°, 3 cm); loss
    0.5·W·L1(C) + 1.0·W·L1(D) ({α,β} TUM setting) (BASELINE.json configs[2])."""
    intr = Intrinsics(525.0, 525.0, 319.5, 239.5, 640, 480)
    scene, poses, kfs, opacity, rng_img = _config_room("tracking", seed, intr, (6.0, 5.0, 3.0), 12, 11)
    # the 11th trajectory pose continues the path; the tracked frame sits half way to it
    p9, p10 = poses[9], poses[10]
    R9, t9 = pose_to_Rt(p9)
    R10, t10 = pose_to_Rt(p10)
    dR = R9.T @ R10
    q = rotmat_to_quat(dR)
    ang = 2 * math.acos(min(1.0, q[0]))
    axis = q[1:] if np.linalg.norm(q[1:]) > 0 else np.array([0, 0, 1.0])
    gt = Rt_to_pose(R9 @ axis_angle_to_rotmat(axis, ang / 2), 0.5 * (t9 + t10))
    d, c = ray_cast(scene, gt, intr, rng_img)
    frame = Frame(d, c, gt)
    rng_p = np.random.Generator(np.random.PCG64([seed, 5]))
    init = perturb_pose(gt, 1.5, 0.03, rng_p)
    cfg = Config("tracking", intr, kfs[:10], opacity[:10], [init], [frame], (0.5, 1.0), "tracking", seed)
    cfg.extra["gt_pose"] = gt
    cfg.extra["iterations"] = 40
    cfg.extra["lr_rot"] = 0.002
    cfg.extra["lr_trans"] = 0.002
    return cfg


def _config4(seed: int) -> Config:
    """Batched mapping: 16 keyframes 640×480 in an 8×6×3 m room with 20 boxes; 8 views =
    keyframes {0,2,…,14} (BASELINE.json configs[3])."""
    intr = Intrinsics(525.0, 525.0, 319.5, 239.5, 640, 480)
    scene, poses, kfs, opacity, _ = _config_room("batched_mapping", seed, intr, (8.0, 6.0, 3.0), 20, 16)
    idx = list(range(0, 16, 2))
    return Config("batched_mapping", intr, kfs, opacity, [kfs[i].pose for i in idx],
                  [kfs[i] for i in idx], (0.8, 1.0), "mapping", seed)


def _config5(seed: int) -> Config:
    """Large: 2×2 floor plan of 6×5×3 m rooms (0.1 m interior walls with 1.0×2.1 m doorways),
    40 boxes, 40 keyframes 1.5 m apart on a ~60 m loop path, 1200×680; 16 views = even
    keyframes (BASELINE.json configs[4])."""
    intr = Intrinsics(600.0, 600.0, 599.5, 339.5, 1200, 680)
    rng_scene = np.random.Generator(np.random.PCG64([seed, 1]))
    rng_img = np.random.Generator(np.random.PCG64([seed, 3]))
    rng_opa = np.random.Generator(np.random.PCG64([seed, 4]))
    X, Y, Z = 12.0, 10.0, 3.0
    th = 0.05
    walls = [
        # wall x = 6 (two segments, each with a doorway)
        ([6 - th, 0.0, 0.0], [6 + th, 2.0, Z]), ([6 - th, 3.0, 0.0], [6 + th, 7.0, Z]),
        ([6 - th, 8.0, 0.0], [6 + th, Y, Z]),
        ([6 - th, 2.0, 2.1], [6 + th, 3.0, Z]), ([6 - th, 7.0, 2.1], [6 + th, 8.0, Z]),
        # wall y = 5
        ([0.0, 5 - th, 0.0], [2.5, 5 + th, Z]), ([3.5, 5 - th, 0.0], [8.5, 5 + th, Z]),
        ([9.5, 5 - th, 0.0], [X, 5 + th, Z]),
        ([2.5, 5 - th, 2.1], [3.5, 5 + th, Z]), ([8.5, 5 - th, 2.1], [9.5, 5 + th, Z]),
    ]
    # loop through the four room centres via the doorways: (3,2.5)->(9,2.5)->(9,7.5)->(3,7.5)
    loop = np.array([[3.0, 2.5], [9.0, 2.5], [9.0, 7.5], [3.0, 7.5]])
    keep = [(x, y, 0.9) for x, y in loop]
    path_pts = []
    for i in range(4):
        a, b = loop[i], loop[(i + 1) % 4]
        for s in np.linspace(0, 1, 25, endpoint=False):
            path_pts.append(a + s * (b - a))
    for (x, y) in path_pts:
        keep.append((x, y, 0.7))
    scene = _room_scene((X, Y, Z), 40, rng_scene, walls=walls, keepout=keep)
    # arc-length parametrisation, 1.5 m between keyframes
    seg = np.concatenate([loop, loop[:1]])
    lens = np.linalg.norm(np.diff(seg, axis=0), axis=1)
    total = float(lens.sum())
    poses = []
    for k in range(40):
        s = (k * 1.5) % total
        i = 0
        while s > lens[i]:
            s -= lens[i]
            i += 1
        d = (seg[i + 1] - seg[i]) / lens[i]
        p = seg[i] + s * d
        yaw = math.atan2(d[1], d[0]) + math.radians(35.0 * math.sin(0.7 * k))
        poses.append(look_pose(np.array([p[0], p[1], 1.5]), yaw, math.radians(-8.0)))
    kfs = []
    for p in poses:
        dpt, c = ray_cast(scene, p, intr, rng_img)
        kfs.append(Frame(dpt, c, p))
    opacity = _sigmoid(rng_opa.normal(size=(40, intr.height, intr.width))).astype(np.float32)
    idx = list(range(0, 32, 2))
    return Config("large", intr, kfs, opacity, [kfs[i].pose for i in idx], [kfs[i] for i in idx],
                  (0.8, 1.0), "mapping", seed)


_BUILDERS = {1: _config1, 2: _config2, 3: _config3, 4: _config4, 5: _config5}


def make_config(which: int, seed: int = 0) -> Config:
    """Build BASELINE.json configs[which-1] deterministically from `seed`."""
    return _BUILDERS[which](seed)


def micro_scene(seed: int, n: int = 12, width: int = 16, height: int = 16) -> dict:
    """A tiny random scene of `n` Gaussians given directly by state (x,y,z,r)/(r,g,b,o) in front
    of an identity-ish camera; used by finite-difference and invariant tests."""
    rng = np.random.Generator(np.random.PCG64([seed, 99]))
    f = 14.0
    intr = Intrinsics(f, f * 1.1, (width - 1) / 2, (height - 1) / 2, width, height)
    z = rng.uniform(1.0, 3.0, size=n)
    u = rng.uniform(1.0, width - 2.0, size=n)
    v = rng.uniform(1.0, height - 2.0, size=n)
    x = (u - intr.cx) * z / intr.fx
    y = (v - intr.cy) * z / intr.fy
    sig_px = rng.uniform(0.8, 2.2, size=n)
    r = sig_px * z / (0.5 * (intr.fx + intr.fy))
    pos_rad = np.stack([x, y, z, r], 1).astype(np.float32)
    col = rng.uniform(0.0, 1.0, size=(n, 3))
    opa = rng.uniform(0.1, 0.9, size=(n, 1))
    col_opa = np.concatenate([col, opa], 1).astype(np.float32)
    q = np.array([1.0, 0.0, 0.0, 0.0]) + rng.normal(0, 0.02, size=4)
    view = np.concatenate([q, rng.normal(0, 0.02, size=3)])
    return {"intr": intr, "pos_rad": pos_rad, "col_opa": col_opa, "view": view}


_CFG_CACHE: dict = {}


def cached_config(which: int, seed: int = 0) -> Config:
    """Process-wide cache of make_config (generation of the large configs takes seconds)."""
    key = (which, seed)
    if key not in _CFG_CACHE:
        _CFG_CACHE[key] = make_config(which, seed)
    return _CFG_CACHE[key]


def pretrack_scene(seed: int = 0) -> dict:
    """A small head-frame selection scene: a 6×5×3 m room with
    12 boxes seen at 96×72 (f = 80) along a 30-frame trajectory (10 cm / 5° steps).  Sections of 5
    frames: section k holds frames [5k, 5k+5); its Gaussians tie frames 5k and 5k+2.  Candidate
    views every N1 = 5 frames (frames 0, 5, …, 25; candidate i belongs to section i).  The head
    frame to track is trajectory frame 29 (ray-cast at ground truth), initialised at GT ∘ (1°, 2 cm)."""
    intr = Intrinsics(80.0, 80.0, 47.5, 35.5, 96, 72)
    scene, poses, kfs, opacity, rng_img = _config_room("pretrack", seed, intr, (6.0, 5.0, 3.0), 12, 30)
    head = kfs[29]
    rng_p = np.random.Generator(np.random.PCG64([seed, 7]))
    init = perturb_pose(head.pose, 1.0, 0.02, rng_p)
    sections = [{"frames": [5 * k, 5 * k + 2], "vis_frames": [5 * k, 5 * k + 2, 5 * k + 4]} for k in range(6)]
    return {"intr": intr, "frames": kfs, "opacity": opacity, "sections": sections, "candidates": list(range(0, 30, 5)),
            "cand_section": [i // 5 for i in range(0, 30, 5)], "head": head, "init": init,
            "gamma": 0.26, "iterations": 8, "lr": 0.002}

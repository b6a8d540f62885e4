"""Pins for the CPU oracle (task rule ③): the oracle is checked against things other than
itself — SPEC worked examples, closed forms, special cases, invariants, brute force on tiny
inputs and central finite differences — so that a dropped term, a wrong sign or index, or a
transposed operand fails at least one of these.  CPU only (`-m "not gpu"`).

Citations: S:n = /root/reference/SPEC.md line n, P:n = PAPER.md line n.
"""
import math

import numpy as np
import pytest

import oracle
from synth.scenes import Intrinsics, cached_config as get_config, micro_scene, perturb_pose

IDENT = np.array([1.0, 0, 0, 0, 0, 0, 0])
MODES = ["f32", "f64"]


def _state(gs):
    """gs: list of (X, Y, Z, r, (cr, cg, cb), o) in world = camera coordinates."""
    pr = np.array([[g[0], g[1], g[2], g[3]] for g in gs], dtype=np.float64)
    co = np.array([[*g[4], g[5]] for g in gs], dtype=np.float64)
    return pr, co


def _intr(f=10.0, W=16, H=16, cx=8.0, cy=8.0, fy=None):
    return Intrinsics(f, f if fy is None else fy, cx, cy, W, H)


# ------------------------------------------------------------------------------ (a1)
@pytest.mark.parametrize("mode", MODES)
def test_back_project_spec_examples(mode):
    """(cx,cy), d=1, identity → (0,0,1); (cx+fx, cy), d=2 → (2,0,2);
    (cx,cy), d=1, translation (0,0,5) → (0,0,6)."""
    intr = Intrinsics(4.0, 4.0, 2.0, 3.0, 8, 6)
    depth = np.zeros((3, 6, 8))
    depth[0, 3, 2] = 1.0
    depth[1, 3, 6] = 2.0
    depth[2, 3, 2] = 1.0
    poses = np.stack([IDENT, IDENT, np.array([1.0, 0, 0, 0, 0, 0, 5.0])])
    rgb = np.full((3, 6, 8, 3), 0.25)
    pr, co, n = oracle.instantiate(depth, rgb, poses, intr, None, 0.5, mode=mode)
    assert n == 3
    g = lambda k, y, x: (k * 6 + y) * 8 + x
    np.testing.assert_allclose(pr[g(0, 3, 2), :3], [0, 0, 1], atol=0)
    np.testing.assert_allclose(pr[g(1, 3, 6), :3], [2, 0, 2], atol=0)
    np.testing.assert_allclose(pr[g(2, 3, 2), :3], [0, 0, 6], atol=0)
    np.testing.assert_allclose(co[g(0, 3, 2)], [0.25, 0.25, 0.25, 0.5])


@pytest.mark.parametrize("mode", MODES)
def test_radius_and_count(mode):
    """d = 2 m, f = 500 → r = 0.004 m; S:440 count = valid pixels; S:442 all-invalid →
    no Gaussians (every slot r = 0)."""
    intr = Intrinsics(500.0, 500.0, 3.5, 2.5, 8, 6)
    rng = np.random.default_rng(1)
    depth = np.where(rng.random((1, 6, 8)) < 0.3, 0.0, 2.0)
    pr, co, n = oracle.instantiate(depth, np.zeros((1, 6, 8, 3)), IDENT[None], intr, mode=mode)
    assert n == int((depth > 0).sum())
    r = pr[:, 3].reshape(6, 8)
    tol = 6e-8 if mode == "f32" else 1e-15   # one fp32 rounding of 2/500
    np.testing.assert_allclose(r[depth[0] > 0], 0.004, rtol=tol)
    assert np.all(pr.reshape(6, 8, 4)[depth[0] == 0] == 0)
    pr0, co0, n0 = oracle.instantiate(np.zeros((1, 6, 8)), np.zeros((1, 6, 8, 3)), IDENT[None], intr, mode=mode)
    assert n0 == 0 and not pr0.any() and not co0.any()


def test_project_back_project_roundtrip():
    """S:75 / S:90: project(back_project(p, d)) = (p, d) within 1e-9 (fp64), random poses."""
    rng = np.random.default_rng(7)
    intr = Intrinsics(525.0, 530.0, 319.5, 239.5, 640, 480)
    K = 4
    depth = rng.uniform(0.5, 5.0, size=(K, 480, 640))
    poses = np.stack([perturb_pose(IDENT, rng.uniform(0, 90), rng.uniform(0, 2), rng) for _ in range(K)])
    pr, co, n = oracle.instantiate(depth, np.zeros((K, 480, 640, 3)), poses, intr, mode="f64")
    for k in range(K):
        sl = slice(k * 480 * 640, (k + 1) * 480 * 640)
        p = oracle.project(pr[sl], poses[k], intr, mode="f64")
        xs, ys = np.meshgrid(np.arange(640), np.arange(480))
        np.testing.assert_allclose(p["proj"][:, 0].reshape(480, 640), xs, atol=1e-9)
        np.testing.assert_allclose(p["proj"][:, 1].reshape(480, 640), ys, atol=1e-9)
        np.testing.assert_allclose(p["proj"][:, 2].reshape(480, 640), depth[k], rtol=1e-12)
        # view-tied self-render: σ = f·(d/f)/d = 1 px (S:140 arithmetic, P:698 r = D/f)
        np.testing.assert_allclose(p["proj"][:, 3], 1.0 * (0.5 * (525 + 530)) / (0.5 * (525 + 530)), rtol=1e-12)


@pytest.mark.parametrize("mode", MODES)
def test_projection_special_cases(mode):
    """identity view → centre (cx, cy), z = depth; behind camera culled;
    r = 0.004, z = 2, f = 500 → σ = 1.0 px.  S:135 near clip 0.01 m; S:127 σ clamp 0.3 px."""
    intr = Intrinsics(500.0, 500.0, 320.0, 240.0, 640, 480)
    pr, _ = _state([(0, 0, 2.0, 0.004, (1, 1, 1), 0.5),
                    (0, 0, -1.0, 0.004, (1, 1, 1), 0.5),
                    (0, 0, 0.01, 0.001, (1, 1, 1), 0.5),
                    (0, 0, 0.0101, 0.001, (1, 1, 1), 0.5),
                    (0, 0, 2.0, 0.0004, (1, 1, 1), 0.5),
                    (0, 0, 2.0, 0.0, (1, 1, 1), 0.5),
                    (1e3, 0, 2.0, 0.004, (1, 1, 1), 0.5)])
    p = oracle.project(pr, IDENT, intr, mode=mode)
    np.testing.assert_allclose(p["proj"][0], [320.0, 240.0, 2.0, 1.0], rtol=1e-7)
    assert p["status"][0] == 1
    np.testing.assert_array_equal(p["rect"][0], [317, 237, 323, 243])   # ±3σ integer rect
    assert p["status"][1] == 0            # behind the camera
    assert p["status"][2] == 0            # z = 0.01 is culled (z ≤ 0.01)
    assert p["status"][3] in (1, 3)       # z = 0.0101 is kept
    assert p["status"][4] == 3 and p["proj"][4, 3] == pytest.approx(0.3, rel=1e-7)   # clamped
    assert p["status"][5] == 0            # invalid slot (r = 0)
    assert p["status"][6] == 0            # footprint entirely outside the image


def test_view_tied_self_render_config1():
    """A keyframe rendered from its own pose puts every centre on its own pixel with σ = 1 px
    (fp32 mode, within fp32 rounding)."""
    c = get_config(1)
    pr, co, n = oracle.instantiate(c.depth_stack(), c.rgb_stack(), c.pose_stack(), c.intr, c.opacity)
    p = oracle.project(pr, c.keyframes[0].pose.astype(np.float32), c.intr)
    xs, ys = np.meshgrid(np.arange(64), np.arange(48))
    assert np.all(p["status"] > 0)
    np.testing.assert_allclose(p["proj"][:, 0].reshape(48, 64), xs, atol=2e-4)
    np.testing.assert_allclose(p["proj"][:, 1].reshape(48, 64), ys, atol=2e-4)
    np.testing.assert_allclose(p["proj"][:, 3], 1.0, rtol=1e-6)


# ------------------------------------------------------------------------------ (a3)
def _brute_tiles(pr, view, intr, mode):
    p = oracle.project(pr, view, intr, mode=mode)
    ntx, nty = (intr.width + 15) // 16, (intr.height + 15) // 16
    lists = [[] for _ in range(ntx * nty)]
    for g in range(len(pr)):
        if not p["status"][g]:
            continue
        x0, y0, x1, y1 = p["rect"][g]
        for ty in range(nty):
            for tx in range(ntx):
                # tile [16tx, 16tx+15] × [16ty, 16ty+15] overlaps the rect?
                if x0 <= 16 * tx + 15 and x1 >= 16 * tx and y0 <= 16 * ty + 15 and y1 >= 16 * ty:
                    z = p["proj"][g, 2]
                    key = np.float32(z).view(np.uint32) if mode == "f32" else z
                    lists[ty * ntx + tx].append((key, g))
    return [[g for _, g in sorted(l)] for l in lists]


@pytest.mark.parametrize("mode", MODES)
def test_tile_lists_brute_force(mode):
    """Brute force over every (tile, Gaussian) pair, sorted by (z bits, gid)."""
    c = get_config(1)
    pr, co, n = oracle.instantiate(c.depth_stack(), c.rgb_stack(), c.pose_stack(), c.intr, c.opacity, mode=mode)
    for view in (c.views[0], c.keyframes[0].pose):
        start, gid = oracle.tile_lists(pr, view, c.intr, mode=mode)
        ref = _brute_tiles(pr, view, c.intr, mode)
        assert start[-1] == sum(len(l) for l in ref) == len(gid)
        for t, l in enumerate(ref):
            assert list(gid[start[t]:start[t + 1]]) == l


def test_tile_lists_equal_depth_tie_break():
    """Equal z → ascending gid (owner frame, pixel index)."""
    intr = _intr(W=32, H=16)
    pr, _ = _state([(0.01 * k, 0.0, 2.0, 0.2, (1, 0, 0), 0.5) for k in range(5)][::-1])
    start, gid = oracle.tile_lists(pr, IDENT, intr)
    for t in range(len(start) - 1):
        l = list(gid[start[t]:start[t + 1]])
        assert l == sorted(l)


# ------------------------------------------------------------------------------ (a4)
@pytest.mark.parametrize("mode", MODES)
def test_single_gaussian_closed_form(mode):
    """One Gaussian centred on pixel (8,8), σ = 1 px: at the centre w = 1 so α = o and
    C = o·c, D = o·z, S = o; one pixel away w = e^{−1/2}."""
    intr = _intr()
    z, o, c = 2.0, 0.6, (0.2, 0.5, 0.9)
    pr, co = _state([(0, 0, z, z / 10.0, c, o)])
    r = oracle.render(pr, co, IDENT, intr, mode=mode)
    tol = 1e-12 if mode == "f64" else 1e-6
    np.testing.assert_allclose(r["color"][8, 8], np.array(c) * o, atol=tol)
    assert r["depth"][8, 8] == pytest.approx(o * z, abs=tol)
    assert r["sil"][8, 8] == pytest.approx(o, abs=tol)
    w1 = math.exp(-0.5)
    assert r["sil"][8, 9] == pytest.approx(o * w1, abs=tol)
    assert r["sil"][9, 9] == pytest.approx(o * math.exp(-1.0), abs=tol)
    # 3σ truncation: pixel (8, 11) is at distance 3 = 3σ (inclusive), (8, 12) at 4 > 3σ
    assert r["sil"][8, 11] == pytest.approx(o * math.exp(-4.5), abs=tol)
    assert r["sil"][8, 12] == 0.0
    assert r["n_comp"][8, 8] == 1 and r["n_comp"][8, 12] == 0


@pytest.mark.parametrize("mode", MODES)
def test_two_gaussians_over_operator(mode):
    """Front-to-back over operator: S = o1 + (1−o1)·o2, C = o1 c1 + (1−o1) o2 c2 — in depth
    order regardless of gid order."""
    intr = _intr()
    o1, o2 = 0.7, 0.4
    c1, c2 = (1.0, 0.0, 0.0), (0.0, 0.0, 1.0)
    for order in (0, 1):
        gs = [(0, 0, 1.0, 0.1, c1, o1), (0, 0, 2.0, 0.2, c2, o2)]
        if order:
            gs = gs[::-1]
        pr, co = _state(gs)
        r = oracle.render(pr, co, IDENT, intr, mode=mode)
        tol = 1e-12 if mode == "f64" else 1e-6
        assert r["sil"][8, 8] == pytest.approx(o1 + (1 - o1) * o2, abs=tol)
        np.testing.assert_allclose(r["color"][8, 8], [o1, 0, (1 - o1) * o2], atol=tol)
        assert r["depth"][8, 8] == pytest.approx(o1 * 1.0 + (1 - o1) * o2 * 2.0, abs=tol)
        assert r["T_final"][8, 8] == pytest.approx((1 - o1) * (1 - o2), abs=tol)


@pytest.mark.parametrize("mode", MODES)
def test_alpha_clamp_and_termination(mode):
    """α = min(o·w, 0.999); T cut-off 1e-4 tested before compositing (reading 8):
    three opaque layers → only the first is composited (T would drop to 1e-6)."""
    intr = _intr()
    c = [(1.0, 0, 0), (0, 1.0, 0), (0, 0, 1.0)]
    pr, co = _state([(0, 0, 1.0 + k, (1.0 + k) / 10, c[k], 1.0) for k in range(3)])
    r = oracle.render(pr, co, IDENT, intr, mode=mode)
    tol = 1e-7 if mode == "f32" else 1e-12
    assert r["sil"][8, 8] == pytest.approx(0.999, abs=tol)
    np.testing.assert_allclose(r["color"][8, 8], [0.999, 0, 0], atol=tol)
    assert r["n_comp"][8, 8] == 1
    # T after two layers: 0.01·0.02 = 2e-4 ≥ 1e-4 → second composited; 0.01·0.005 < 1e-4 → not
    for a2, expect_n in ((0.98, 2), (0.995, 1)):
        pr, co = _state([(0, 0, 1.0, 0.1, c[0], 0.99), (0, 0, 2.0, 0.2, c[1], a2)])
        r = oracle.render(pr, co, IDENT, intr, mode=mode)
        assert r["n_comp"][8, 8] == expect_n
        s = 0.99 + (0.01 * a2 if expect_n == 2 else 0.0)
        assert r["sil"][8, 8] == pytest.approx(s, abs=1e-6)
        assert r["T_final"][8, 8] >= 1e-4


@pytest.mark.parametrize("mode", MODES)
def test_alpha_floor(mode):
    """α < 1/255 is skipped (north_star (4)): o = 0.0039 renders nothing, o = 0.004 renders."""
    intr = _intr()
    for o, expect in ((0.0039, 0.0), (0.004, 0.004)):
        pr, co = _state([(0, 0, 2.0, 0.2, (1, 1, 1), o)])
        r = oracle.render(pr, co, IDENT, intr, mode=mode)
        assert r["sil"][8, 8] == pytest.approx(expect, abs=1e-9)


@pytest.mark.parametrize("mode", MODES)
def test_truncation_beats_floor(mode):
    """σ = 0.6 px, o = 1: at distance 1.7 px (< 3σ) w = e^{−1.7²/0.72} ≈ 0.018 renders; at
    1.9 px (> 3σ = 1.8) w ≈ 0.0067 > 1/255 would pass the floor but is truncated."""
    intr = Intrinsics(10.0, 10.0, 8.0, 8.0, 16, 16)
    z = 2.0
    for dxp, expect in ((1.7, math.exp(-1.7 ** 2 / 0.72)), (1.9, 0.0)):
        X = -dxp * z / 10.0                        # centre at u = 8 − dxp
        pr, co = _state([(X, 0.0, z, 0.6 * z / 10.0, (1, 1, 1), 1.0)])
        r = oracle.render(pr, co, IDENT, intr, mode=mode)
        assert r["sil"][8, 8] == pytest.approx(expect, abs=1e-6)


def _random_render(seed, mode="f64", n=30):
    m = micro_scene(seed, n=n)
    r = oracle.render(m["pos_rad"], m["col_opa"], m["view"], m["intr"], mode=mode)
    return m, r


@pytest.mark.parametrize("seed", range(8))
def test_render_invariants(seed):
    """S:121 S ∈ [0,1], S = 0 ⇒ C = 0 and D = 0; S = 1 − T_final exactly in fp64 (Σ αT of the
    over operator telescopes); T_final ≥ 1e-4 (cut-off); zero opacities → background."""
    m, r = _random_render(seed)
    S = r["sil"]
    assert S.min() >= 0 and S.max() <= 1
    z = S == 0
    assert np.all(r["color"][z] == 0) and np.all(r["depth"][z] == 0)
    np.testing.assert_allclose(S, 1.0 - r["T_final"], atol=1e-12)
    assert r["T_final"].min() >= 1e-4
    co0 = m["col_opa"].copy()
    co0[:, 3] = 0.0
    r0 = oracle.render(m["pos_rad"], co0, m["view"], m["intr"], mode="f64")
    assert not r0["color"].any() and not r0["depth"].any() and not r0["sil"].any()


@pytest.mark.parametrize("seed", range(4))
def test_silhouette_monotone_in_opacity(seed):
    """raising one opacity never lowers a pixel's silhouette — up to the 1e-4
    transmittance cut-off, which can end a pixel one Gaussian earlier (S ≤ 1 − 1e-4 then)."""
    m, r = _random_render(seed, n=20)
    for g in range(0, 20, 3):
        co = m["col_opa"].copy().astype(np.float64)
        co[g, 3] = min(1.0, co[g, 3] + 0.3)
        r2 = oracle.render(m["pos_rad"], co, m["view"], m["intr"], mode="f64")
        assert np.all(r2["sil"] >= r["sil"] - 1e-4)


@pytest.mark.parametrize("seed", range(3))
def test_permutation_invariance(seed):
    """permuting the inputs (distinct depths) gives bit-identical images."""
    m = micro_scene(seed, n=25)
    perm = np.random.default_rng(seed).permutation(25)
    for mode in MODES:
        a = oracle.render(m["pos_rad"], m["col_opa"], m["view"], m["intr"], mode=mode)
        b = oracle.render(m["pos_rad"][perm], m["col_opa"][perm], m["view"], m["intr"], mode=mode)
        for k in ("color", "depth", "sil", "T_final"):
            assert np.array_equal(a[k], b[k])


def _brute_render(pr, co, view, intr):
    """Naive per-pixel compositing over ALL Gaussians sorted by (z, gid) — no tiles."""
    p = oracle.project(pr, view, intr, mode="f64")
    order = sorted([g for g in range(len(pr)) if p["status"][g]], key=lambda g: (p["proj"][g, 2], g))
    H, W = intr.height, intr.width
    out = np.zeros((H, W, 5))
    for y in range(H):
        for x in range(W):
            T = 1.0
            acc = np.zeros(5)
            for g in order:
                u, v, z, s = p["proj"][g]
                x0, y0, x1, y1 = p["rect"][g]
                if not (x0 <= x <= x1 and y0 <= y <= y1):
                    continue
                d2 = (x - u) ** 2 + (y - v) ** 2
                if d2 > 9 * s * s:
                    continue
                a = min(co[g, 3] * math.exp(-0.5 * d2 / (s * s)), 0.999)
                if a < 1 / 255:
                    continue
                if T * (1 - a) < 1e-4:
                    break
                acc += a * T * np.array([co[g, 0], co[g, 1], co[g, 2], z, 1.0])
                T *= 1 - a
            out[y, x] = acc
    return out


@pytest.mark.parametrize("seed", range(3))
def test_brute_force_per_pixel_render(seed):
    """the tile-list renderer equals a naive per-pixel full-sort compositor (fp64)."""
    m = micro_scene(seed, n=30)
    r = oracle.render(m["pos_rad"], m["col_opa"], m["view"], m["intr"], mode="f64")
    b = _brute_render(m["pos_rad"].astype(np.float64), m["col_opa"].astype(np.float64), m["view"], m["intr"])
    np.testing.assert_allclose(r["color"], b[..., :3], atol=1e-12)
    np.testing.assert_allclose(r["depth"], b[..., 3], atol=1e-12)
    np.testing.assert_allclose(r["sil"], b[..., 4], atol=1e-12)


def test_f32_mode_matches_f64_mode_config1():
    """The fp32-decision oracle and the fp64 oracle agree to fp32 accuracy on config 1,
    wherever the fp32 near-threshold flag is clear."""
    c = get_config(1)
    a_pr, a_co, _ = oracle.instantiate(c.depth_stack(), c.rgb_stack(), c.pose_stack(), c.intr, c.opacity, mode="f32")
    b_pr, b_co, _ = oracle.instantiate(c.depth_stack(), c.rgb_stack(), c.pose_stack(), c.intr, c.opacity, mode="f64")
    a = oracle.render(a_pr, a_co, c.views[0], c.intr, mode="f32")
    b = oracle.render(b_pr, b_co, c.views[0], c.intr, mode="f64")
    ok = ~a["flags"]
    assert (a["n_comp"][ok] == b["n_comp"][ok]).mean() > 0.999
    np.testing.assert_allclose(a["sil"][ok], b["sil"][ok], atol=2e-5)
    np.testing.assert_allclose(a["depth"][ok], b["depth"][ok], atol=1e-4)


# ------------------------------------------------------------------------------ (a5)
def _fd_check(m, seed, eps=1e-6, n_params=None):
    pr = m["pos_rad"].astype(np.float64)
    co = m["col_opa"].astype(np.float64)
    view = np.asarray(m["view"], dtype=np.float64)
    intr = m["intr"]
    rng = np.random.default_rng(seed)
    H, W = intr.height, intr.width
    lC, lD, lS = rng.normal(size=(H, W, 3)), rng.normal(size=(H, W)), rng.normal(size=(H, W))

    def L(pr_, co_, view_):
        r = oracle.render(pr_, co_, view_, intr, mode="f64")
        return (r["color"] * lC).sum() + (r["depth"] * lD).sum() + (r["sil"] * lS).sum(), r["trace"]

    _, t0 = L(pr, co, view)
    g = oracle.render_bwd(pr, co, view, intr, lC, lD, lS, mode="f64")
    checked = skipped = 0
    worst = 0.0

    def one(f, analytic):
        nonlocal checked, skipped, worst
        (lp, tp), (lm, tm) = f(eps), f(-eps)
        if not (np.array_equal(tp, t0) and np.array_equal(tm, t0)):
            skipped += 1          # a discrete decision changed inside ±ε (S:224 boundary)
            return
        fd = (lp - lm) / (2 * eps)
        err = abs(fd - analytic) / max(abs(analytic), 1e-3)
        worst = max(worst, err)
        checked += 1

    N = len(pr) if n_params is None else n_params
    for i in range(N):
        for j in range(4):
            def f(e, i=i, j=j):
                a = co.copy(); a[i, j] += e
                return L(pr, a, view)
            one(f, g["d_col_opa"][i, j])

        def f(e, i=i):
            a = pr.copy(); a[i, 3] += e
            return L(a, co, view)
        one(f, g["d_radius"][i])
    for j in range(7):
        def f(e, j=j):
            a = view.copy(); a[j] += e
            return L(pr, co, a)
        one(f, g["d_pose"][j])
    return checked, skipped, worst


@pytest.mark.parametrize("seed", range(10))
def test_gradients_central_differences(seed):
    """S:205 / S:218: analytic gradients of a random linear functional of (C, D, S) match
    central finite differences for colour, opacity, radius and the 7 pose parameters
    (ambient quaternion + translation).  fp64, ε = 1e-6; parameters whose ±ε runs change a
    discrete decision (3σ boundary, floor, cut-off) are skipped and must stay rare."""
    m = micro_scene(seed, n=12)
    checked, skipped, worst = _fd_check(m, seed)
    assert checked >= 60 and skipped <= 3
    assert worst < 1e-5


def test_gradients_central_differences_config1():
    """Same check on config 1 (64×48, 3,072 view-tied Gaussians, perturbed pose), first 40
    Gaussians + the pose."""
    c = get_config(1)
    pr, co, _ = oracle.instantiate(c.depth_stack(), c.rgb_stack(), c.pose_stack(), c.intr, c.opacity, mode="f64")
    # pick Gaussians near the centre (well inside the image) so their footprints render
    m = {"pos_rad": pr, "col_opa": co, "view": c.views[0], "intr": c.intr}
    sel = np.arange(20 * 64 + 20, 20 * 64 + 60)
    order = np.concatenate([sel, np.setdiff1d(np.arange(len(pr)), sel)])
    m["pos_rad"], m["col_opa"] = pr[order], co[order]
    checked, skipped, worst = _fd_check(m, 5, n_params=40)
    assert checked >= 150 and skipped <= 10
    assert worst < 1e-4


def test_zero_upstream_and_zero_opacity():
    """zero upstream → all-zero bundle; an opacity-0 Gaussian gets d_color = 0."""
    m = micro_scene(11, n=15)
    co = m["col_opa"].astype(np.float64).copy()
    co[3, 3] = 0.0
    H, W = m["intr"].height, m["intr"].width
    g = oracle.render_bwd(m["pos_rad"], co, m["view"], m["intr"], np.zeros((H, W, 3)), np.zeros((H, W)),
                          np.zeros((H, W)), mode="f64")
    assert not g["d_col_opa"].any() and not g["d_radius"].any() and not g["d_pose"].any()
    rng = np.random.default_rng(0)
    g = oracle.render_bwd(m["pos_rad"], co, m["view"], m["intr"], rng.normal(size=(H, W, 3)),
                          rng.normal(size=(H, W)), rng.normal(size=(H, W)), mode="f64")
    assert not g["d_col_opa"][3, :3].any()


def test_single_gaussian_gradient_closed_form():
    """At the centre pixel of a lone Gaussian: ∂C/∂c = o·I, ∂S/∂o = 1, ∂D/∂z-depth = o."""
    intr = _intr()
    pr, co = _state([(0, 0, 2.0, 0.2, (0.3, 0.3, 0.3), 0.6)])
    H, W = 16, 16
    for ch in range(3):
        gC = np.zeros((H, W, 3)); gC[8, 8, ch] = 1.0
        g = oracle.render_bwd(pr, co, IDENT, intr, gC, None, None, mode="f64")
        expect = np.zeros(4); expect[ch] = 0.6; expect[3] = 0.3   # ∂C_ch/∂o = w·c = 0.3
        np.testing.assert_allclose(g["d_col_opa"][0], expect, atol=1e-12)
    gS = np.zeros((H, W)); gS[8, 8] = 1.0
    g = oracle.render_bwd(pr, co, IDENT, intr, None, None, gS, mode="f64")
    assert g["d_col_opa"][0, 3] == pytest.approx(1.0, abs=1e-12)
    # the centre pixel's silhouette is stationary in u, v, σ (w has a maximum there)
    np.testing.assert_allclose(g["d_geom"][0, :3], 0.0, atol=1e-12)


def test_loss_at_optimum_gives_zero_gradient():
    """Target rendered from the same parameters → every residual is exactly 0 → with
    sgn(0) = 0 every gradient is exactly 0 (SURVEY §8(c) pin for a5)."""
    c = get_config(1)
    pr, co, _ = oracle.instantiate(c.depth_stack(), c.rgb_stack(), c.pose_stack(), c.intr, c.opacity)
    r = oracle.render(pr, co, c.views[0], c.intr)
    loss, gC, gD, gS, fl = oracle.l1_upstream(r["color"], r["depth"], r["sil"], r["color"], r["depth"],
                                               None, 1.0, 0.5, 0, 0, 0)
    assert loss == 0.0 and not gC.any() and not gD.any()
    g = oracle.render_bwd(pr, co, c.views[0], c.intr, gC, gD, gS)
    assert not g["d_col_opa"].any() and not g["d_radius"].any() and not g["d_pose"].any()


# ------------------------------------------------------------------------------ losses
def test_l1_loss_examples():
    """S:256-258 masked_l1: a = b → 0; constant difference 0.1, full mask → 0.1; empty mask → 0
    with zero gradient.  S:281: α = 0.5, β = 0.025, unit colour error, zero depth error → 0.5.
    S:292 linearity in the weights."""
    H, W = 4, 5
    rng = np.random.default_rng(0)
    C = rng.random((H, W, 3)); D = rng.uniform(1, 2, (H, W)); S = np.ones((H, W))
    loss, *_ = oracle.l1_upstream(C, D, S, C, D, None, 1, 1, 0, 0, 1)
    assert loss == 0.0
    loss, gC, gD, _, _ = oracle.l1_upstream(C, D + 0.1, S, C, D, None, 0, 1, 0, 0, 1)
    assert loss == pytest.approx(0.1, rel=1e-12)
    np.testing.assert_allclose(gD, 1.0 / (H * W))
    loss, gC, gD, _, _ = oracle.l1_upstream(C, D, S, C, np.zeros((H, W)), None, 0, 1, 0, 0, 1)
    assert loss == 0.0 and not gD.any()
    # Replica tracking weights on a full W mask: per-pixel ‖·‖₁ colour error of 1, depth 0
    loss, *_ = oracle.l1_upstream(C + 1.0 / 3.0, D, S, C, D, None, 0.5, 0.025, 1, 1, 1)
    assert loss == pytest.approx(0.5, rel=1e-12)
    # linearity in the weights
    l1, gC1, gD1, *_ = oracle.l1_upstream(C, D, S, C[::-1].copy(), D[::-1].copy(), None, 0.3, 0.7, 0, 0, 0)
    l2, gC2, gD2, *_ = oracle.l1_upstream(C, D, S, C[::-1].copy(), D[::-1].copy(), None, 0.6, 1.4, 0, 0, 0)
    assert l2 == pytest.approx(2 * l1, rel=1e-12)
    np.testing.assert_allclose(gC2, 2 * gC1)
    np.testing.assert_allclose(gD2, 2 * gD1)


def test_tracking_mask_semantics():
    """P:146 / S:336: W = valid ∧ S > 0.99 ∧ vis; with color_mask_mode = 1 only W pixels count."""
    H, W = 2, 3
    C = np.zeros((H, W, 3)); tC = np.ones((H, W, 3))
    D = np.ones((H, W)); tD = np.array([[1.5, 0.0, 1.5], [1.5, 1.5, 1.5]])
    S = np.array([[1.0, 1.0, 0.5], [1.0, 1.0, 1.0]])
    vis = np.array([[1, 1, 1], [1, 0, 1]], dtype=np.uint8)
    loss, gC, gD, _, _ = oracle.l1_upstream(C, D, S, tC, tD, vis, 1.0, 1.0, 1, 1, 0)
    Wm = np.array([[1, 0, 0], [1, 0, 1]], dtype=bool)
    assert loss == pytest.approx(Wm.sum() * (3 * 1.0 + 0.5))
    assert np.all((gC != 0).any(-1) == Wm) and np.all((gD != 0) == Wm)


# ------------------------------------------------------------------------------ f1 (head-frame BA)
def _two_keyframe_scene(seed, W=14, H=12, K=2):
    """K keyframes of a noisy tilted plane (depth 1.5–2.5 m), a view near keyframe 0."""
    rng = np.random.default_rng(seed)
    intr = Intrinsics(12.0, 12.5, (W - 1) / 2, (H - 1) / 2, W, H)
    poses, depth = [], []
    for k in range(K):
        poses.append(perturb_pose(np.array([1.0, 0, 0, 0, 0, 0, 0]), 3.0 * k, 0.05 * k, rng))
        xs = np.arange(W)[None, :]
        depth.append(1.5 + 0.05 * xs + 0.03 * np.arange(H)[:, None] + rng.normal(0, 0.01, (H, W)))
    depth = np.stack(depth)
    rgb = rng.uniform(0, 1, (K, H, W, 3))
    opa = 1 / (1 + np.exp(-rng.normal(size=(K, H, W))))
    view = perturb_pose(poses[0], 1.0, 0.02, rng)
    return intr, np.stack(poses), depth, rgb, opa, view


@pytest.mark.parametrize("seed", range(3))
def test_keyframe_pose_gradient_central_differences(seed):
    """P:248-250 (head-frame bundle adjustment): dL/d(keyframe pose) through the view-tied centres
    X_w = R_k X_k + t_k, from the per-Gaussian dL/dX_w, against central finite differences of a
    random linear functional of (C, D, S) re-instantiating the keyframes (fp64, ε = 1e-6)."""
    intr, poses, depth, rgb, opa, view = _two_keyframe_scene(seed)
    H, W = intr.height, intr.width
    rng = np.random.default_rng(100 + seed)
    lC, lD, lS = rng.normal(size=(H, W, 3)), rng.normal(size=(H, W)), rng.normal(size=(H, W))

    def L(ps):
        pr, co, _ = oracle.instantiate(depth, rgb, ps, intr, opa, mode="f64")
        r = oracle.render(pr, co, view, intr, mode="f64")
        return (r["color"] * lC).sum() + (r["depth"] * lD).sum() + (r["sil"] * lS).sum(), r["trace"]

    pr, co, _ = oracle.instantiate(depth, rgb, poses, intr, opa, mode="f64")
    g = oracle.render_bwd(pr, co, view, intr, lC, lD, lS, mode="f64")
    ana = oracle.keyframe_pose_grad(depth, poses, intr, g["d_pos"])
    _, t0 = L(poses)
    eps, checked, worst = 1e-6, 0, 0.0
    for k in range(len(poses)):
        for j in range(7):
            pp, pm = poses.copy(), poses.copy()
            pp[k, j] += eps
            pm[k, j] -= eps
            (lp, tp), (lm, tm) = L(pp), L(pm)
            if not (np.array_equal(tp, t0) and np.array_equal(tm, t0)):
                continue
            fd = (lp - lm) / (2 * eps)
            worst = max(worst, abs(fd - ana[k, j]) / max(abs(ana[k, j]), 1e-3))
            checked += 1
    assert checked >= 12 and worst < 1e-5, (checked, worst)


def test_view_tied_pose_invariance():
    """Rendering keyframe k's own Gaussians from keyframe k's own pose does not depend on that
    pose (the centres move with the camera): the view-pose gradient and the owner-pose
    gradient cancel exactly, d_view + d_kf = 0, and a rigid motion of both leaves the image."""
    intr, poses, depth, rgb, opa, _ = _two_keyframe_scene(3, K=1)
    H, W = intr.height, intr.width
    rng = np.random.default_rng(7)
    lC, lD, lS = rng.normal(size=(H, W, 3)), rng.normal(size=(H, W)), rng.normal(size=(H, W))
    view = poses[0]
    pr, co, _ = oracle.instantiate(depth, rgb, poses, intr, opa, mode="f64")
    g = oracle.render_bwd(pr, co, view, intr, lC, lD, lS, mode="f64")
    kf = oracle.keyframe_pose_grad(depth, poses, intr, g["d_pos"])[0]
    scale = np.abs(g["d_pose"]).max()
    assert scale > 1e-3
    np.testing.assert_allclose(g["d_pose"] + kf, 0.0, atol=1e-8 * max(scale, 1.0))


# ------------------------------------------------------------------------------ f2 (SSIM of Eq. 2)
def test_ssim_identity_and_symmetry():
    """L_S(x, x) = 0 with zero gradient (SSIM's maximum, "a = b → SSIM 1, L_S 0");
    SSIM is symmetric in its arguments; τ scales value and gradient (linearity in weights)."""
    rng = np.random.default_rng(0)
    x, y = rng.uniform(size=(14, 17, 3)), rng.uniform(size=(14, 17, 3))
    l0, g0 = oracle.ssim_loss(x, x, tau=0.2)
    assert l0 == 0.0 and np.abs(g0).max() < 1e-15
    a, _ = oracle.ssim_loss(x, y, tau=0.2)
    b, _ = oracle.ssim_loss(y, x, tau=0.2)
    assert a > 0 and abs(a - b) < 1e-14
    c, gc = oracle.ssim_loss(x, y, tau=0.4)
    _, ga = oracle.ssim_loss(x, y, tau=0.2)
    assert abs(c - 2 * a) < 1e-14 and np.allclose(gc, 2 * ga, rtol=0, atol=1e-15)


def test_ssim_constant_images_closed_form():
    """Constant images a, b: at pixels whose 11×11 window lies inside the image the window
    weights sum to 1 and both variances vanish, so SSIM = (2ab + C1)/(a² + b² + C1)
    ("a constant 0, b constant 1 → C1/(1 + C1)")."""
    H, W = 16, 18
    for a, b in ((0.0, 1.0), (0.3, 0.7), (0.5, 0.5)):
        _, _, smap = oracle.ssim_loss(np.full((H, W, 3), a), np.full((H, W, 3), b), want_map=True)
        C1 = 0.01 ** 2
        ref = (2 * a * b + C1) / (a * a + b * b + C1)
        np.testing.assert_allclose(smap[5:H - 5, 5:W - 5], ref, rtol=1e-12)


def test_ssim_gradient_central_differences():
    """Gradient of τ·L_S w.r.t. the render against central differences (fp64, ε = 1e-6) at
    every pixel of a 12×13 image."""
    rng = np.random.default_rng(1)
    x, y = rng.uniform(size=(12, 13, 3)), rng.uniform(size=(12, 13, 3))
    _, g = oracle.ssim_loss(x, y, tau=0.2)
    eps = 1e-6
    worst = 0.0
    for idx in np.ndindex(*x.shape):
        xp, xm = x.copy(), x.copy()
        xp[idx] += eps
        xm[idx] -= eps
        fd = (oracle.ssim_loss(xp, y)[0] - oracle.ssim_loss(xm, y)[0]) / (2 * eps)
        worst = max(worst, abs(fd - g[idx]) / max(abs(g[idx]), 1e-6))
    assert worst < 1e-5


# ------------------------------------------------------------------------------ f4 (densification)
def test_densify_special_cases():
    """silhouette ≡ 1 → no new Gaussians; silhouette ≡ 0 (empty section) → exactly
    init_gaussians' valid slots, in row-major order; otherwise the new set is {valid ∧ S < 0.5}
    (strict), each initialised as init_gaussians."""
    rng = np.random.default_rng(4)
    H, W = 9, 11
    intr = Intrinsics(10.0, 11.0, 5.0, 4.0, W, H)
    depth = np.where(rng.random((H, W)) < 0.2, 0.0, rng.uniform(0.5, 3.0, (H, W)))
    rgb = rng.random((H, W, 3))
    pose = perturb_pose(IDENT, 5.0, 0.1, rng)
    opa = rng.random((H, W))
    pr, co = oracle.densify(depth, rgb, pose, intr, np.ones((H, W)), 0.5, opa)
    assert len(pr) == 0
    pr, co = oracle.densify(depth, rgb, pose, intr, np.zeros((H, W)), 0.5, opa)
    ipr, ico, n = oracle.instantiate(depth[None], rgb[None], pose[None], intr, opa[None])
    valid = depth.reshape(-1) > 0
    assert len(pr) == n and np.array_equal(pr, ipr[valid]) and np.array_equal(co, ico[valid])
    sil = rng.random((H, W))
    sil[0, 0] = 0.5                      # exactly at the threshold: covered (strict <)
    depth[0, 0] = 1.0
    pr, co = oracle.densify(depth, rgb, pose, intr, sil, 0.5, opa)
    ipr, ico, _ = oracle.instantiate(depth[None], rgb[None], pose[None], intr, opa[None])
    sel = (depth.reshape(-1) > 0) & (sil.reshape(-1) < 0.5)
    assert not sel[0] and len(pr) == sel.sum()
    assert np.array_equal(pr, ipr[sel]) and np.array_equal(co, ico[sel])


# ------------------------------------------------------------------------------ f3 (visibility)
def _plane_frame(W=24, H=18, f=20.0, seed=0):
    rng = np.random.default_rng(seed)
    intr = Intrinsics(f, f, (W - 1) / 2, (H - 1) / 2, W, H)
    xs, ys = np.meshgrid(np.arange(W), np.arange(H))
    depth = 2.0 + 0.02 * xs + 0.01 * ys
    return intr, depth, rng


@pytest.mark.parametrize("mode", MODES)
def test_visibility_special_cases(mode):
    """P:186 / S:313-322: a frame's own back-projected points are visible to itself (SPEC
    "self-consistency"), a depth band of 1% decides (z = 1.02·d → not visible, 1.005·d →
    visible), points outside the reference frustum are not visible, and the section mask is the
    union of the per-reference masks."""
    intr, depth, rng = _plane_frame()
    pose = IDENT
    own = oracle.visibility(depth, pose, depth[None], pose[None], intr, mode=mode)
    assert own.mean() > 0.99
    far = oracle.visibility(depth, pose, (depth / 1.02)[None], pose[None], intr, mode=mode)
    assert not far.any()
    near = oracle.visibility(depth, pose, (depth / 1.005)[None], pose[None], intr, mode=mode)
    assert near.mean() > 0.99
    away = np.array([0.0, 0.0, 1.0, 0.0, 0, 0, 0])          # 180° about y: looking backwards
    assert not oracle.visibility(depth, pose, depth[None], away[None], intr, mode=mode).any()
    # fronto-parallel wall 2 m away seen from a camera 30 cm to the side: partial overlap
    wall = np.full_like(depth, 2.0)
    shifted = np.array([1.0, 0, 0, 0, 0.3, 0.0, 0.0])
    m_a = oracle.visibility(wall, pose, wall[None], shifted[None], intr, mode=mode)
    u_ref = np.arange(intr.width) - 0.3 * intr.fx / 2.0      # each column's wall point in the shifted view
    assert m_a[:, (u_ref > 0.5) & (u_ref < intr.width - 1.5)].all()
    assert not m_a[:, u_ref < -0.5].any()
    m_b = oracle.visibility(wall, pose, (wall / 1.005)[None], pose[None], intr, mode=mode)
    m_c = oracle.visibility(wall, pose, (wall / 1.02)[None], pose[None], intr, mode=mode)
    m_ab = oracle.visibility(wall, pose, np.stack([wall, wall / 1.02]), np.stack([shifted, pose]), intr, mode=mode)
    assert 0 < m_a.mean() < 1 and m_b.all() and not m_c.any() and np.array_equal(m_ab, m_a | m_c)
    loose = oracle.visibility(depth, pose, (depth / 1.015)[None], pose[None], intr, tol=0.02, mode=mode)
    assert loose.mean() > 0.99          # monotone in the tolerance


# ------------------------------------------------------------------------------ round-2 pins
def test_rotation_known_values():
    """The pose convention pinned by known rotations, not by round trips (camera-to-world,
    unit quaternion (w,x,y,z); 90° z-rotations compose to 180°).  With the Hamilton
    convention q = (cos θ/2, 0, 0, sin θ/2) rotates by θ about +z, so for θ = 90° the camera's +x
    axis maps to world +y (a transposed R would map it to −y); q = (cos 45°, sin 45°, 0, 0)
    maps camera +y to world +z; q = (0, 0, 0, 1) (two 90° z-turns) maps +x to −x.  Pixel
    (cx+fx, cy) at d = 2 is X_c = (2, 0, 2), pixel (cx, cy+fy) at d = 2 is X_c = (0, 2, 2)
    (S:66); the world point is R·X_c + t with t = (1, 2, 3)."""
    c, s = math.cos(math.pi / 4), math.sin(math.pi / 4)
    intr = Intrinsics(4.0, 4.0, 2.0, 3.0, 8, 6)
    cases = [  # (pose, pixel, world)
        ([c, 0, 0, s, 1, 2, 3], (6, 3), (1.0, 4.0, 5.0)),     # +x → +y
        ([c, 0, 0, s, 1, 2, 3], (2, 7 - 4), (1.0, 2.0, 5.0)),  # principal ray (0,0,2) → (0,0,2)
        ([0, 0, 0, 1, 1, 2, 3], (6, 3), (-1.0, 2.0, 5.0)),    # 180° about z: +x → −x
        ([c, 0, s, 0, 1, 2, 3], (6, 3), (3.0, 2.0, 1.0)),     # 90° about y: +x → −z, +z → +x
    ]
    for pose, (x, y), world in cases:
        if world is None:
            continue
        for mode in MODES:
            depth = np.zeros((1, 6, 8))
            depth[0, y, x] = 2.0
            pr, _, n = oracle.instantiate(depth, np.zeros((1, 6, 8, 3)), np.array([pose]), intr, mode=mode)
            np.testing.assert_allclose(pr[y * 8 + x, :3], world, atol=1e-6, err_msg=f"{pose} {mode}")
    # camera +y → world +z under a 90° turn about +x: pixel (cx, cy + fy/2) at d = 2 is X_c = (0, 1, 2)
    # → R·X_c = (0, −2, 1) (y → z, z → −y), + t = (1, 0, 4)
    intr2 = Intrinsics(4.0, 4.0, 2.0, 1.0, 8, 6)
    for mode in MODES:
        depth = np.zeros((1, 6, 8))
        depth[0, 3, 2] = 2.0
        pr, _, _ = oracle.instantiate(depth, np.zeros((1, 6, 8, 3)), np.array([[c, s, 0, 0, 1, 2, 3]]), intr2, mode=mode)
        np.testing.assert_allclose(pr[3 * 8 + 2, :3], (1.0, 0.0, 4.0), atol=1e-6)
    # and the view transform is its inverse: projecting that world point from the same pose
    # gives back the pixel and the depth (S:75 round trip through a non-trivial rotation)
    p = oracle.project(np.array([[1.0, 0.0, 4.0, 0.01]]), np.array([c, s, 0, 0, 1, 2, 3]), intr2, mode="f64")
    np.testing.assert_allclose(p["proj"][0, :3], (2.0, 3.0, 2.0), atol=1e-12)


def test_pose_adam_spec_examples():
    """S:207-215 (adam_step): zero gradient → parameters unchanged; constant gradient g, first step
    → Δ = −lr·g/(|g| + ε) ≈ −lr·sign(g) (bias correction makes m̂ = g, v̂ = g²), and the same
    again on the second step; the quaternion is renormalised after every step (|q| = 1 within
    1e-9); separate rates for rotation and translation."""
    q = np.array([0.9, 0.1, -0.3, 0.2])
    pose0 = np.concatenate([q / np.linalg.norm(q), [0.5, -1.0, 2.0]])
    p, st = oracle.pose_adam(pose0, np.zeros(7), np.zeros(15), 0.01, 0.02)
    np.testing.assert_allclose(p, pose0, atol=1e-15)
    assert st[14] == 1.0
    g = np.array([0.0, 0.0, 0.0, 0.0, 3.0, -0.5, 1e-3])
    p1, st1 = oracle.pose_adam(pose0, g, np.zeros(15), 0.01, 0.02)
    np.testing.assert_allclose(p1[4:] - pose0[4:], -0.02 * g[4:] / (np.abs(g[4:]) + 1e-8), rtol=1e-12)
    np.testing.assert_allclose(p1[:4], pose0[:4], atol=1e-15)        # zero rotation gradient
    p2, _ = oracle.pose_adam(p1, g, st1, 0.01, 0.02)
    np.testing.assert_allclose(p2[4:] - p1[4:], -0.02 * g[4:] / (np.abs(g[4:]) + 1e-8), rtol=1e-9)
    rng = np.random.default_rng(0)
    p, st = pose0.copy(), np.zeros(15)
    for _ in range(20):
        p, st = oracle.pose_adam(p, rng.normal(size=7), st, 0.05, 0.01)
        assert abs(np.linalg.norm(p[:4]) - 1.0) < 1e-9
    # a rotation-only gradient moves q by ≈ lr per component before renormalisation
    gq = np.array([1.0, -1.0, 0.0, 0.0, 0, 0, 0])
    p3, _ = oracle.pose_adam(np.array([1.0, 0, 0, 0, 0, 0, 0]), gq, np.zeros(15), 0.01, 0.02)
    raw = np.array([1.0 - 0.01, 0.01, 0.0, 0.0])
    np.testing.assert_allclose(p3[:4], raw / np.linalg.norm(raw), atol=1e-9)
    np.testing.assert_allclose(p3[4:], 0.0, atol=0)


def _brute_render_vec(pr, co, view, intr):
    """Naive compositing over ALL Gaussians in (z, gid) order, every pixel at once."""
    p = oracle.project(pr, view, intr, mode="f64")
    order = sorted([g for g in range(len(pr)) if p["status"][g]], key=lambda g: (p["proj"][g, 2], g))
    H, W = intr.height, intr.width
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64)
    T = np.ones((H, W))
    alive = np.ones((H, W), dtype=bool)
    acc = np.zeros((H, W, 5))
    for g in order:
        u, v, z, s = p["proj"][g]
        x0, y0, x1, y1 = p["rect"][g]
        inr = (xs >= x0) & (xs <= x1) & (ys >= y0) & (ys <= y1)
        d2 = (xs - u) ** 2 + (ys - v) ** 2
        a = np.minimum(co[g, 3] * np.exp(-0.5 * d2 / (s * s)), 0.999)
        el = alive & inr & (d2 <= 9 * s * s) & (a >= 1 / 255)
        Tn = T * (1 - a)
        stop = el & (Tn < 1e-4)
        alive &= ~stop
        comp = el & ~stop
        acc[comp] += (a * T)[comp][:, None] * np.array([co[g, 0], co[g, 1], co[g, 2], z, 1.0])
        T = np.where(comp, Tn, T)
    return acc


def test_tiled_equals_naive_1000_trials():
    """S:166 and SPEC acceptance 2: the tiled renderer (tile lists, per-tile depth order) equals
    a naive per-pixel compositor over all Gaussians within 1e-5 on ≥ 1000 random scenes at
    16×16 … 32×32 (fp64 oracle mode; ragged sizes included)."""
    worst = 0.0
    for t in range(1000):
        rng = np.random.default_rng(1000 + t)
        W, H = int(rng.integers(16, 33)), int(rng.integers(16, 33))
        m = micro_scene(t, n=int(rng.integers(1, 31)), width=W, height=H)
        pr, co = m["pos_rad"].astype(np.float64), m["col_opa"].astype(np.float64)
        r = oracle.render(pr, co, m["view"], m["intr"], mode="f64")
        b = _brute_render_vec(pr, co, m["view"], m["intr"])
        err = max(np.abs(r["color"] - b[..., :3]).max(), np.abs(r["depth"] - b[..., 3]).max(),
                  np.abs(r["sil"] - b[..., 4]).max())
        worst = max(worst, err)
        assert err <= 1e-5, (t, err)
    assert worst <= 1e-12


def test_gradients_central_differences_100_scenes():
    """S:218 / SPEC acceptance 1: analytic gradients (colour, opacity, radius, the 7 pose
    parameters) against central finite differences on ≥ 100 random micro-scenes (16×16, ≤ 30
    Gaussians), fp64.  Parameters whose ±ε runs change a discrete decision are skipped."""
    total = skipped_all = 0
    worst_all = 0.0
    for seed in range(100, 200):
        m = micro_scene(seed, n=5 + seed % 26)
        checked, skipped, worst = _fd_check(m, seed)
        total += checked
        skipped_all += skipped
        worst_all = max(worst_all, worst)
        assert worst < 1e-5, (seed, worst)
    assert total >= 100 * 40 and skipped_all <= 0.02 * total, (total, skipped_all)

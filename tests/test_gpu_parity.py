"""GPU parity: the CUDA path through the C ABI against the CPU oracle, element by element, on
the same seeded inputs (task rule ③).  Bars (BASELINE.json north_star):
  * instantiation and tile lists / sort order: bit-exact;
  * colour, depth, silhouette: within 1e-4 absolute (fp32) on every pixel the oracle does not
    flag as near a decision threshold ("near-threshold flags");
  * gradients: within 1e-3 relative or 1e-5 absolute on every Gaussian not evaluated at a
    flagged pixel (plus, for the handful of sums that cancel by κ > 1e3, the fp32 summation
    floor 16·2⁻²⁴·Σ|terms| — DESIGN.md §3 R23 — counted and capped); the pose gradient within
    1e-3 of its norm.
"""
import ctypes

import numpy as np
import pytest

import oracle
from synth.scenes import Intrinsics, cached_config, micro_scene
from vtgs_testlib import check_grads, close, combine_allow, flip_allowance, gpu_instantiate, oracle_instantiate, report, view32

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def vt():
    from paper_2506_02741_b200 import vtgs
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return vtgs


def _renderer(vt, cfg, **kw):
    return vt.Renderer(0, cfg.n_slots, cfg.intr.width, cfg.intr.height, **kw)


def _view(cfg):
    return view32(cfg.views[0])


def _loss_of(cfg):
    wc, wd = cfg.loss_weights
    mode = 1 if cfg.mode == "tracking" else 0
    return dict(w_color=wc, w_depth=wd, color_mask_mode=mode, depth_mask_mode=mode, normalize=0)


def _render_gpu(vt, R, cfg, pos_rad, col_opa, view=None):
    """Forward; the view pose and the output images are kept alive on the renderer because the
    context reads them again in the backward (vtgs.h: they must stay valid until render_bwd)."""
    v = vt.pose_tensor(_view(cfg) if view is None else view, "cuda")
    out = R.render_fwd(pos_rad, col_opa, v, cfg.intr)
    R._keep = (v, out, pos_rad, col_opa)
    torch.cuda.synchronize()
    return v, out


# ------------------------------------------------------------------------------ (a1)
@pytest.mark.parametrize("which", [1, 2, 3])
def test_instantiate_bitexact(vt, which):
    """(a1) bit-exact slots, and the valid-slot count n_valid equal to the oracle's."""
    cfg = cached_config(which)
    R = _renderer(vt, cfg)
    nv = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    pr, co = R.instantiate(torch.from_numpy(cfg.depth_stack()).cuda(), torch.from_numpy(cfg.rgb_stack()).cuda(),
                           vt.pose_tensor(cfg.pose_stack(), "cuda"), cfg.intr, torch.from_numpy(cfg.opacity).cuda(),
                           n_valid=nv)
    opr, oco, on = oracle.instantiate(cfg.depth_stack(), cfg.rgb_stack(), cfg.pose_stack(), cfg.intr, cfg.opacity)
    assert np.array_equal(pr.cpu().numpy(), opr.astype(np.float32))
    assert np.array_equal(co.cpu().numpy(), oco.astype(np.float32))
    assert int(nv.item()) == on


# ------------------------------------------------------------------------------ (a2)/(a3)
@pytest.mark.parametrize("which,view", [(1, "view"), (1, "kf"), (2, "view"), (3, "view"), (4, "view")])
def test_tile_lists_bitexact(vt, which, view):
    cfg = cached_config(which)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    v = view32(cfg.keyframes[0].pose) if view == "kf" else _view(cfg)
    _render_gpu(vt, R, cfg, pr, co, v)
    start, gid = R.export_tiles(cfg.intr)
    opr, _ = oracle_instantiate(cfg)
    ostart, ogid = oracle.tile_lists(opr, v, cfg.intr)
    assert np.array_equal(start, ostart), "tile offsets differ"
    assert np.array_equal(gid.astype(np.int64), ogid), "sorted tile lists differ"
    st = R.stats()
    assert st["n_pairs"] == len(ogid) and st["max_tile"] == int(np.diff(ostart).max())


def test_tile_lists_micro_scenes(vt):
    """Random micro scenes (non-unit q, fx ≠ fy, σ 0.8–2.2 px, many overlaps)."""
    for seed in range(10):
        m = micro_scene(seed, n=200, width=45, height=37)
        R = vt.Renderer(0, 200, 45, 37)
        pr = torch.from_numpy(m["pos_rad"]).cuda()
        co = torch.from_numpy(m["col_opa"]).cuda()
        v = vt.pose_tensor(view32(m["view"]), "cuda")
        R.render_fwd(pr, co, v, m["intr"])
        start, gid = R.export_tiles(m["intr"])
        ostart, ogid = oracle.tile_lists(m["pos_rad"], view32(m["view"]), m["intr"])
        assert np.array_equal(start, ostart) and np.array_equal(gid.astype(np.int64), ogid)


@pytest.mark.parametrize("case", ["equal_depth", "two_depths", "long_lists", "very_long_lists", "equal_depth_long"])
def test_tile_lists_sort_paths(vt, case):
    """The per-tile sort's paths, bit-exact against the oracle: equal or nearly equal depths (a
    bucket larger than the bucket sort takes → radix hand-off, ties broken by gid), and lists
    longer than the on-chip bucket sort (> 4096 entries per tile: depth-bucketed into chunks that
    are sorted on chip, several chunks per tile for the very long lists).  The sub-lists of the
    long tiles are checked through the forward render against the oracle's."""
    rng = np.random.Generator(np.random.PCG64([7, {"equal_depth": 0, "two_depths": 1, "long_lists": 2,
                                                   "very_long_lists": 3, "equal_depth_long": 4}[case]]))
    W, H = 40, 36
    intr = Intrinsics(30.0, 30.0, (W - 1) / 2, (H - 1) / 2, W, H)
    n = {"long_lists": 20000, "very_long_lists": 60000, "equal_depth_long": 30000}.get(case, 6000)
    if case in ("equal_depth", "equal_depth_long"):   # the long one: radix sort on global scratch
        z = np.full(n, 2.0)
    elif case == "two_depths":
        z = np.where(rng.random(n) < 0.5, 2.0, np.nextafter(np.float32(2.0), np.float32(3.0)))
    else:
        z = rng.uniform(1.0, 4.0, size=n)
    u = rng.uniform(0.0, W - 1.0, size=n)
    v = rng.uniform(0.0, H - 1.0, size=n)
    x = (u - intr.cx) * z / intr.fx
    y = (v - intr.cy) * z / intr.fy
    r = rng.uniform(0.8, 2.5, size=n) * z / intr.fx
    pos_rad = np.stack([x, y, z, r], 1).astype(np.float32)
    col_opa = np.concatenate([rng.random((n, 3)), rng.uniform(0.01, 0.2, (n, 1))], 1).astype(np.float32)
    view = np.array([1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0])
    R = vt.Renderer(0, n, W, H)
    pr = torch.from_numpy(pos_rad).cuda()
    co = torch.from_numpy(col_opa).cuda()
    pv = vt.pose_tensor(view32(view), "cuda")
    out = R.render_fwd(pr, co, pv, intr)
    start, gid = R.export_tiles(intr)
    ostart, ogid = oracle.tile_lists(pos_rad, view32(view), intr)
    assert np.array_equal(start, ostart) and np.array_equal(gid.astype(np.int64), ogid)
    if case == "long_lists":
        assert np.diff(ostart).max() > 4096
    if case == "very_long_lists":
        assert np.diff(ostart).max() > 3 * 4096
    if case == "equal_depth_long":
        assert np.diff(ostart).max() > 8192
    ref = oracle.render(pos_rad, col_opa, view32(view), intr)
    _check_images(out, ref, ref["flags"], max_flagged=2e-2)
    # gradients through the same (chunked / radix-sorted) sub-lists: the backward walks the long
    # tiles' lists back to front from the forward's exact composited masks
    rg = np.random.default_rng(5)
    gC = rg.normal(size=(H, W, 3)).astype(np.float32)
    gD = rg.normal(size=(H, W)).astype(np.float32)
    gS = rg.normal(size=(H, W)).astype(np.float32)
    R._keep = (pv, out, pr, co)
    want = vt.VTGS_GRAD_ALL
    dco = torch.zeros((n, 4), device="cuda")
    drad = torch.zeros(n, device="cuda")
    dpose = torch.zeros(7, device="cuda")
    R.render_bwd(want, d_col_opa=dco, d_radius=drad, d_pose=dpose, dL_dcolor=torch.from_numpy(gC).cuda(),
                 dL_ddepth=torch.from_numpy(gD).cuda(), dL_dsil=torch.from_numpy(gS).cuda())
    torch.cuda.synchronize()
    reft = oracle.render(pos_rad, col_opa, view32(view), intr, want_tainted=True)
    g = oracle.render_bwd(pos_rad, col_opa, view32(view), intr, gC, gD, gS, want_allow=True)
    check_grads(vt, want, dco.cpu().numpy().astype(np.float64), drad.cpu().numpy().astype(np.float64),
                dpose.cpu().numpy().astype(np.float64), g, reft["tainted"], allow=combine_allow(g),
                name=f"sort path {case}", cap=2e-2)


# ------------------------------------------------------------------------------ (a4)
def _check_images(out, ref, flags, atol=1e-4, max_flagged=5e-3):
    color, depth, sil = (t.cpu().numpy().astype(np.float64) for t in out)
    ok = ~flags
    assert flags.mean() < max_flagged, f"too many flagged pixels: {flags.sum()}"
    for name, g, r in (("color", color[ok], ref["color"][ok]), ("depth", depth[ok], ref["depth"][ok]),
                       ("sil", sil[ok], ref["sil"][ok])):
        good = np.abs(g - r) <= atol
        assert good.all(), report(name, good, g, r)


@pytest.mark.parametrize("which", [1, 2, 3])
def test_forward_parity(vt, which):
    cfg = cached_config(which)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    _, out = _render_gpu(vt, R, cfg, pr, co)
    opr, oco = oracle_instantiate(cfg)
    ref = oracle.render(opr, oco, _view(cfg), cfg.intr)
    _check_images(out, ref, ref["flags"])
    st = R.stats()
    assert st["overflow"] == 0
    assert st["n_pairs"] == ref["stats"][2]
    # composited / evaluated pair counts agree up to the flagged pixels
    assert abs(st["e_comp"] - ref["stats"][1]) <= max(10, 2e-4 * ref["stats"][1])
    assert abs(st["e_eval"] - ref["stats"][0]) <= max(10, 2e-4 * ref["stats"][0])


def test_forward_parity_config4_sampled_rows(vt):
    """Config 4 (16 keyframes, 4.9M slots) at full size, oracle on sampled row bands."""
    cfg = cached_config(4)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    opr, oco = oracle_instantiate(cfg)
    for k in (0, 3):
        v = view32(cfg.views[k])
        _, out = _render_gpu(vt, R, cfg, pr, co, v)
        for r0 in (0, 200, 464):
            ref = oracle.render(opr, oco, v, cfg.intr, rows=(r0, r0 + 16))
            sl = slice(r0, r0 + 16)
            sub = tuple(t[sl] for t in out)
            _check_images(sub, {kk: ref[kk][sl] for kk in ("color", "depth", "sil")}, ref["flags"][sl])


@pytest.mark.parametrize("seed", range(6))
def test_forward_parity_micro_ragged(vt, seed):
    """Ragged image sizes (not multiples of 16), dense overlaps, σ clamp cases."""
    W, H = [(45, 37), (17, 16), (16, 17), (33, 1), (1, 40), (100, 61)][seed]
    m = micro_scene(seed, n=300, width=max(W, 4), height=max(H, 4))
    intr = Intrinsics(m["intr"].fx, m["intr"].fy, W / 2 - 0.25, H / 2 - 0.25, W, H) \
        if min(W, H) > 1 else Intrinsics(14.0, 15.0, W / 2, H / 2, W, H)
    R = vt.Renderer(0, 300, W, H)
    pr = torch.from_numpy(m["pos_rad"]).cuda()
    co = torch.from_numpy(m["col_opa"]).cuda()
    v = view32(m["view"])
    vv = vt.pose_tensor(v, "cuda")
    out = R.render_fwd(pr, co, vv, intr)
    ref = oracle.render(m["pos_rad"], m["col_opa"], v, intr)
    _check_images(out, ref, ref["flags"])


# ------------------------------------------------------------------------------ (a5)
def _oracle_grads(cfg, opr, oco, v, gC, gD, gS, flip=None):
    """Oracle gradients for the upstream (gC, gD, gS); the taint comes from the forward's decision
    near-ties only; `flip` (L1 sgn near-ties) becomes a per-Gaussian allowance."""
    ref = oracle.render(opr, oco, v, cfg.intr, want_tainted=True)
    g = oracle.render_bwd(opr, oco, v, cfg.intr, gC, gD, gS, want_allow=True)
    allow = combine_allow(g, None if flip is None else flip_allowance(opr, oco, v, cfg.intr, flip))
    return ref, g, allow


def _check_grads(want, dco, drad, dpose, g, tainted, vt, learn=None, allow=None, name=""):
    return check_grads(vt, want, dco, drad, dpose, g, tainted, allow=allow, learn=learn, name=name)


def _run_bwd(vt, R, cfg, want, n, **kw):
    dco = torch.zeros((n, 4), device="cuda")
    drad = torch.zeros(n, device="cuda")
    dpose = torch.zeros(7, device="cuda")
    R.render_bwd(want, d_col_opa=dco, d_radius=drad, d_pose=dpose, **kw)
    torch.cuda.synchronize()
    return dco.cpu().numpy().astype(np.float64), drad.cpu().numpy().astype(np.float64), \
        dpose.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("which", [1, 2, 3])
def test_backward_parity_upstream(vt, which):
    """Explicit per-pixel upstream gradients (a seeded random linear functional of C, D, S)."""
    cfg = cached_config(which)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    _render_gpu(vt, R, cfg, pr, co)
    H, W = cfg.intr.height, cfg.intr.width
    rng = np.random.default_rng(which)
    gC = rng.normal(size=(H, W, 3)).astype(np.float32)
    gD = rng.normal(size=(H, W)).astype(np.float32)
    gS = rng.normal(size=(H, W)).astype(np.float32)
    want = vt.VTGS_GRAD_ALL
    dco, drad, dpose = _run_bwd(vt, R, cfg, want, cfg.n_slots, dL_dcolor=torch.from_numpy(gC).cuda(),
                                dL_ddepth=torch.from_numpy(gD).cuda(), dL_dsil=torch.from_numpy(gS).cuda())
    opr, oco = oracle_instantiate(cfg)
    ref, g, allow = _oracle_grads(cfg, opr, oco, _view(cfg), gC, gD, gS)
    _check_grads(want, dco, drad, dpose, g, ref["tainted"], vt, allow=allow, name=f"upstream config {which}")


@pytest.mark.parametrize("which", [1, 2, 3])
def test_backward_pose_only_upstream(vt, which):
    """Pose-only backward (the tracking kernel, no per-Gaussian reduction) with explicit
    upstream gradients: d_pose against the oracle's, attribute buffers untouched."""
    cfg = cached_config(which)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    _render_gpu(vt, R, cfg, pr, co)
    H, W = cfg.intr.height, cfg.intr.width
    rng = np.random.default_rng(10 + which)
    gC = rng.normal(size=(H, W, 3)).astype(np.float32)
    gD = rng.normal(size=(H, W)).astype(np.float32)
    gS = rng.normal(size=(H, W)).astype(np.float32)
    dco, drad, dpose = _run_bwd(vt, R, cfg, vt.VTGS_GRAD_POSE, cfg.n_slots, dL_dcolor=torch.from_numpy(gC).cuda(),
                                dL_ddepth=torch.from_numpy(gD).cuda(), dL_dsil=torch.from_numpy(gS).cuda())
    assert not dco.any() and not drad.any()
    opr, oco = oracle_instantiate(cfg)
    ref, g, allow = _oracle_grads(cfg, opr, oco, _view(cfg), gC, gD, gS)
    _check_grads(vt.VTGS_GRAD_POSE, dco, drad, dpose, g, ref["tainted"], vt, allow=allow, name=f"pose-only config {which}")


@pytest.mark.parametrize("which", [1, 2, 3])
def test_backward_parity_fused_l1(vt, which):
    """The config's own objective: masked L1 of Eq. 1 (tracking) / L1 terms of Eq. 2 (mapping),
    sum form (SURVEY §8(c) pin note), fused into the backward."""
    cfg = cached_config(which)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    _render_gpu(vt, R, cfg, pr, co)
    tg = cfg.targets[0]
    L = _loss_of(cfg)
    want = {"full": vt.VTGS_GRAD_ALL, "mapping": vt.VTGS_GRAD_ATTR, "tracking": vt.VTGS_GRAD_POSE}[cfg.mode]
    loss_out = torch.zeros(1, device="cuda")
    dco, drad, dpose = _run_bwd(vt, R, cfg, want, cfg.n_slots, loss=dict(
        target_rgb=torch.from_numpy(tg.rgb).cuda(), target_depth=torch.from_numpy(tg.depth).cuda(), **L),
        loss_out=loss_out)
    opr, oco = oracle_instantiate(cfg)
    v = _view(cfg)
    img = oracle.render(opr, oco, v, cfg.intr)
    loss, gC, gD, gS, lflags, flip = oracle.l1_upstream(img["color"], img["depth"], img["sil"], tg.rgb, tg.depth,
                                                         None, L["w_color"], L["w_depth"], L["color_mask_mode"],
                                                         L["depth_mask_mode"], 0, want_flip=True)
    assert abs(float(loss_out.item()) - loss) <= 1e-4 * abs(loss) + 1e-6
    ref, g, allow = _oracle_grads(cfg, opr, oco, v, gC, gD, gS, flip=flip)
    _check_grads(want, dco, drad, dpose, g, ref["tainted"], vt, allow=allow, name=f"fused L1 config {which}")


@pytest.mark.parametrize("which", [4, 5])
def test_backward_parity_long_lists_full_size(vt, which):
    """Gradient parity on the workloads whose tiles exceed the on-chip sort (configs 4 and 5: tile
    lists up to ~7k and ~58k entries, chunked / radix sort paths) at full size, through the
    config's own mapping objective (L1 terms of Eq. 2, sum form): one view of config 4
    (16 keyframes 640×480, 4.9M slots) and one of config 5 (40 keyframes 1200×680, 32.6M slots)."""
    cfg = cached_config(which)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    v = view32(cfg.views[0])
    _render_gpu(vt, R, cfg, pr, co, v)
    st = R.stats()
    print(f"[long lists config {which}] P = {st['n_pairs']}, longest tile list {st['max_tile']}")
    assert st["overflow"] == 0 and st["max_tile"] > 4096, st
    tg = cfg.targets[0]
    wc, wd = cfg.loss_weights
    want = vt.VTGS_GRAD_ATTR
    dco, drad, dpose = _run_bwd(vt, R, cfg, want, cfg.n_slots, loss=dict(
        target_rgb=torch.from_numpy(tg.rgb).cuda(), target_depth=torch.from_numpy(tg.depth).cuda(), w_color=wc,
        w_depth=wd))
    del pr, co
    opr, oco = oracle_instantiate(cfg)
    img = oracle.render(opr, oco, v, cfg.intr)
    _, gC, gD, gS, _, flip = oracle.l1_upstream(img["color"], img["depth"], img["sil"], tg.rgb, tg.depth, None,
                                                wc, wd, 0, 0, 0, want_flip=True)
    ref, g, allow = _oracle_grads(cfg, opr, oco, v, gC, gD, gS, flip=flip)
    _check_grads(want, dco, drad, dpose, g, ref["tainted"], vt, allow=allow, name=f"long lists config {which}")


@pytest.mark.parametrize("which", [1, 2])
def test_deterministic_attribute_gradients(vt, which):
    """VTGS_GRAD_DETERMINISTIC (fixed merge order): two runs give bit-identical
    attribute gradients, they agree with the float-atomic path to fp32 summation noise, and they
    pass the oracle's gradient bar (config 1 checked against the oracle)."""
    cfg = cached_config(which)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    _render_gpu(vt, R, cfg, pr, co)
    tg = cfg.targets[0]
    L = dict(target_rgb=torch.from_numpy(tg.rgb).cuda(), target_depth=torch.from_numpy(tg.depth).cuda(),
             **_loss_of(cfg))
    det = vt.VTGS_GRAD_ATTR | vt.VTGS_GRAD_DETERMINISTIC
    runs = [_run_bwd(vt, R, cfg, det, cfg.n_slots, loss=L) for _ in range(2)]
    fl = _run_bwd(vt, R, cfg, vt.VTGS_GRAD_ATTR, cfg.n_slots, loss=L)
    assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][1], runs[1][1])
    for a, b in ((runs[0][0], fl[0]), (runs[0][1], fl[1])):
        assert np.allclose(a, b, rtol=1e-4, atol=1e-6)
    if which == 1:
        opr, oco = oracle_instantiate(cfg)
        v = _view(cfg)
        img = oracle.render(opr, oco, v, cfg.intr)
        Lo = _loss_of(cfg)
        _, gC, gD, gS, _, flip = oracle.l1_upstream(img["color"], img["depth"], img["sil"], tg.rgb, tg.depth, None,
                                                    Lo["w_color"], Lo["w_depth"], Lo["color_mask_mode"],
                                                    Lo["depth_mask_mode"], 0, want_flip=True)
        ref, g, allow = _oracle_grads(cfg, opr, oco, v, gC, gD, gS, flip=flip)
        _check_grads(vt.VTGS_GRAD_ATTR, runs[0][0], runs[0][1], None, g, ref["tainted"], vt, allow=allow,
                     name="deterministic merge config 1")


def test_backward_learn_range_and_accumulate(vt):
    """Only gids in [learn_begin, learn_end) get attribute gradients; gradients
    accumulate (+=) across calls (multi-view mapping is a loop)."""
    cfg = cached_config(1)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    _render_gpu(vt, R, cfg, pr, co)
    H, W = cfg.intr.height, cfg.intr.width
    rng = np.random.default_rng(3)
    gC = torch.from_numpy(rng.normal(size=(H, W, 3)).astype(np.float32)).cuda()
    lo, hi = 700, 2100
    dco, drad, _ = _run_bwd(vt, R, cfg, vt.VTGS_GRAD_ATTR, cfg.n_slots, dL_dcolor=gC, learn=(lo, hi))
    opr, oco = oracle_instantiate(cfg)
    ref, g, allow = _oracle_grads(cfg, opr, oco, _view(cfg), gC.cpu().numpy(), None, None)
    _check_grads(vt.VTGS_GRAD_ATTR, dco, drad, None, g, ref["tainted"], vt, learn=(lo, hi), allow=allow,
                 name="learn range")
    acc = torch.zeros((cfg.n_slots, 4), device="cuda")
    accr = torch.zeros(cfg.n_slots, device="cuda")
    R.render_bwd(vt.VTGS_GRAD_ATTR, d_col_opa=acc, d_radius=accr, dL_dcolor=gC)
    R.render_bwd(vt.VTGS_GRAD_ATTR, d_col_opa=acc, d_radius=accr, dL_dcolor=gC)
    one = torch.zeros((cfg.n_slots, 4), device="cuda")
    R.render_bwd(vt.VTGS_GRAD_ATTR, d_col_opa=one, d_radius=torch.zeros_like(accr), dL_dcolor=gC)
    torch.cuda.synchronize()
    assert torch.allclose(acc, 2 * one, rtol=1e-6, atol=1e-7)


# ------------------------------------------------------------------------------ invariants on GPU
def test_loss_at_optimum_zero_gradient(vt):
    """Target = the GPU's own render → every residual is exactly 0 → all gradients exactly 0."""
    cfg = cached_config(1)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    v, (C, D, S) = _render_gpu(vt, R, cfg, pr, co)
    tC, tD = C.clone(), D.clone()
    dco, drad, dpose = _run_bwd(vt, R, cfg, vt.VTGS_GRAD_ALL, cfg.n_slots,
                                loss=dict(target_rgb=tC, target_depth=tD, w_color=1.0, w_depth=0.5))
    assert not dco.any() and not drad.any() and not dpose.any()


def test_deterministic_forward_and_pose(vt):
    cfg = cached_config(3)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    tg = cfg.targets[0]
    L = dict(target_rgb=torch.from_numpy(tg.rgb).cuda(), target_depth=torch.from_numpy(tg.depth).cuda(),
             **_loss_of(cfg))
    outs = []
    for _ in range(2):
        _, img = _render_gpu(vt, R, cfg, pr, co)
        dp = torch.zeros(7, device="cuda")
        R.render_bwd(vt.VTGS_GRAD_POSE, d_pose=dp, loss=L)
        torch.cuda.synchronize()
        outs.append([t.clone() for t in img] + [dp.clone()])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_zero_opacity_background(vt):
    cfg = cached_config(1)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    co[:, 3] = 0.0
    _, (C, D, S) = _render_gpu(vt, R, cfg, pr, co)
    assert not C.any() and not D.any() and not S.any()


# ------------------------------------------------------------------------------ edge cases
def test_edge_empty_and_invalid(vt):
    intr = Intrinsics(60.0, 60.0, 32.0, 24.0, 64, 48)
    R = vt.Renderer(0, 64 * 48, 64, 48)
    v = vt.pose_tensor([1, 0, 0, 0, 0, 0, 0], "cuda")
    e = torch.zeros((0, 4), device="cuda")
    C, D, S = R.render_fwd(e, e, v, intr, N=0)
    torch.cuda.synchronize()
    assert not C.any() and not D.any() and not S.any()
    dp = torch.zeros(7, device="cuda")
    R.render_bwd(vt.VTGS_GRAD_POSE, d_pose=dp, dL_dcolor=torch.ones((48, 64, 3), device="cuda"))
    torch.cuda.synchronize()
    assert not dp.any()
    # all-invalid depth → every slot r = 0 → empty render
    depth = torch.zeros((1, 48, 64), device="cuda")
    rgb = torch.rand((1, 48, 64, 3), device="cuda")
    pr, co = R.instantiate(depth, rgb, v, intr)
    assert not pr.any() and not co.any()
    C, D, S = R.render_fwd(pr, co, v, intr)
    torch.cuda.synchronize()
    assert not S.any()
    # everything behind the camera → culled
    depth = torch.full((1, 48, 64), 2.0, device="cuda")
    pr, co = R.instantiate(depth, rgb, v, intr)
    back = vt.pose_tensor([0, 0, 1, 0, 0, 0, 0], "cuda")   # 180° about y: looks the other way
    C, D, S = R.render_fwd(pr, co, back, intr)
    torch.cuda.synchronize()
    assert not S.any() and R.stats()["n_pairs"] == 0


def test_edge_single_gaussian_closed_form(vt):
    intr = Intrinsics(10.0, 10.0, 8.0, 8.0, 16, 16)
    R = vt.Renderer(0, 1, 16, 16)
    pr = torch.tensor([[0.0, 0.0, 2.0, 0.2]], device="cuda")
    co = torch.tensor([[0.2, 0.5, 0.9, 0.6]], device="cuda")
    v = vt.pose_tensor([1, 0, 0, 0, 0, 0, 0], "cuda")
    C, D, S = R.render_fwd(pr, co, v, intr)
    torch.cuda.synchronize()
    assert S[8, 8].item() == pytest.approx(0.6, abs=1e-6)
    assert D[8, 8].item() == pytest.approx(1.2, abs=1e-6)
    assert S[8, 9].item() == pytest.approx(0.6 * np.exp(-0.5), abs=1e-6)
    assert S[8, 12].item() == 0.0


def test_edge_errors(vt):
    intr = Intrinsics(60.0, 60.0, 32.0, 24.0, 64, 48)
    R = vt.Renderer(0, 3072, 64, 48, max_pairs=100)
    v = vt.pose_tensor([1, 0, 0, 0, 0, 0, 0], "cuda")
    with pytest.raises(vt.VtgsError) as e:
        R.render_bwd(vt.VTGS_GRAD_POSE, d_pose=torch.zeros(7, device="cuda"),
                     dL_dcolor=torch.zeros((48, 64, 3), device="cuda"))
    assert e.value.status == vt.VTGS_ERR_STATE
    bad = Intrinsics(60.0, 60.0, 64.0, 24.0, 64, 48)   # cx not inside (0, W)
    e4 = torch.zeros((1, 4), device="cuda")
    with pytest.raises(vt.VtgsError) as e:
        R.render_fwd(e4, e4, v, bad)
    assert e.value.status == vt.VTGS_ERR_INVALID_ARG
    big = Intrinsics(60.0, 60.0, 32.0, 24.0, 65, 48)
    with pytest.raises(vt.VtgsError) as e:
        R.render_fwd(e4, e4, v, big)
    assert e.value.status == vt.VTGS_ERR_SHAPE
    # more Gaussians than the context holds → VTGS_ERR_CAPACITY (instantiate and render)
    with pytest.raises(vt.VtgsError) as e:
        R.instantiate(torch.zeros((2, 48, 64), device="cuda"), torch.zeros((2, 48, 64, 3), device="cuda"),
                      vt.pose_tensor(np.tile([1.0, 0, 0, 0, 0, 0, 0], (2, 1)), "cuda"), intr)
    assert e.value.status == vt.VTGS_ERR_CAPACITY
    e5 = torch.zeros((3073, 4), device="cuda")
    with pytest.raises(vt.VtgsError) as e:
        R.render_fwd(e5, e5, v, intr)
    assert e.value.status == vt.VTGS_ERR_CAPACITY
    # capacity: 3,072 Gaussians need > 100 pairs → deferred VTGS_ERR_CAPACITY, empty render
    cfg = cached_config(1)
    pr, co = gpu_instantiate(R, cfg)
    C, D, S = R.render_fwd(pr, co, vt.pose_tensor(_view(cfg), "cuda"), cfg.intr)
    with pytest.raises(vt.VtgsError) as e:
        R.check()
    assert e.value.status == vt.VTGS_ERR_CAPACITY
    assert not S.any()
    # the host-buffer step reports the same overflow instead of returning an empty render's loss
    hr = torch.zeros((48, 64, 3)).pin_memory()
    hd = torch.zeros((48, 64)).pin_memory()
    dco = torch.zeros((3072, 4), device="cuda")
    drad = torch.zeros(3072, device="cuda")
    with pytest.raises(vt.VtgsError) as e:
        R.step_host(pr, co, np.asarray(_view(cfg), dtype=np.float32), cfg.intr, hr, hd, 1.0, 1.0, 0, 0, 0,
                    vt.VTGS_GRAD_ATTR, (0, 3072), (C, D, S), dco, drad)
    assert e.value.status == vt.VTGS_ERR_CAPACITY


def test_edge_max_image_size_and_all_layers(vt):
    """Maximum context size exactly, and long tile lists through the global-memory sort path
    (> 4096 entries per tile)."""
    W, H = 48, 32
    intr = Intrinsics(40.0, 40.0, 23.5, 15.5, W, H)
    K = 64                              # 64 stacked fronto-parallel layers → ~64·(16+6)² per tile
    R = vt.Renderer(0, K * W * H, W, H)
    depth = torch.linspace(1.0, 3.0, K, device="cuda")[:, None, None].expand(K, H, W).contiguous()
    rgb = torch.rand((K, H, W, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    poses = vt.pose_tensor(np.tile([1, 0, 0, 0, 0, 0, 0], (K, 1)), "cuda")
    opa = torch.full((K, H, W), 0.05, device="cuda")
    pr, co = R.instantiate(depth, rgb, poses, intr, opa)
    v = view32([1, 0.01, -0.01, 0, 0.01, 0, 0])
    out = R.render_fwd(pr, co, vt.pose_tensor(v, "cuda"), intr)
    st = R.stats()
    assert st["max_tile"] > 4096
    start, gid = R.export_tiles(intr)
    opr, oco, _ = oracle.instantiate(depth.cpu().numpy(), rgb.cpu().numpy(), np.tile([1, 0, 0, 0, 0, 0, 0], (K, 1)),
                                     intr, opa.cpu().numpy())
    ostart, ogid = oracle.tile_lists(opr, v, intr)
    assert np.array_equal(start, ostart) and np.array_equal(gid.astype(np.int64), ogid)
    ref = oracle.render(opr, oco, v, intr)
    # 64 uniform low-opacity layers end every pixel near the 1e-4 cut-off at once, so the
    # near-threshold flag legitimately covers a few percent of this scene
    _check_images(out, ref, ref["flags"], max_flagged=0.05)


# ------------------------------------------------------------------------------ tracking loop
def test_tracking_loop_graph_matches_eager_and_converges(vt):
    """Config 3: 40 iterations of fwd + bwd(pose) + device Adam; the CUDA-graph capture gives
    the same pose as eager launches, and the pose error shrinks."""
    cfg = cached_config(3)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    tg = cfg.targets[0]
    L = dict(target_rgb=torch.from_numpy(tg.rgb).cuda(), target_depth=torch.from_numpy(tg.depth).cuda(),
             w_color=0.5, w_depth=1.0, color_mask_mode=1, depth_mask_mode=1, normalize=1)
    iters = cfg.extra["iterations"]

    def run(graph: bool):
        pose = vt.pose_tensor(_view(cfg), "cuda")
        state = torch.zeros(16, device="cuda")
        dp = torch.zeros(7, device="cuda")
        out = (torch.empty((480, 640, 3), device="cuda"), torch.empty((480, 640), device="cuda"),
               torch.empty((480, 640), device="cuda"))

        def body(stream=None):
            for _ in range(iters):
                R.render_fwd(pr, co, pose, cfg.intr, out=out, stream=stream)
                R.render_bwd(vt.VTGS_GRAD_POSE, d_pose=dp, loss=L, stream=stream)
                R.pose_adam_step(pose, dp, state, cfg.extra["lr_rot"], cfg.extra["lr_trans"], stream=stream)
        if graph:
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                body(stream=s)
            pose.copy_(vt.pose_tensor(_view(cfg), "cuda"))
            state.zero_()
            g.replay()
        else:
            body()
        torch.cuda.synchronize()
        return pose.cpu().numpy()[0]

    pe = run(False)
    pg = run(True)
    assert np.array_equal(pe, pg)
    gt = cfg.extra["gt_pose"]
    init = _view(cfg)
    assert np.linalg.norm(pe[4:] - gt[4:]) < np.linalg.norm(init[4:] - gt[4:])


def test_mapping_step_graph_matches_eager(vt):
    """The bench replays the mapping step (zero grads + fwd + fused L1 + bwd) from one CUDA graph:
    the graph gives the same images and loss bit for bit and the same gradients (float atomics:
    equal up to summation order) as eager launches."""
    from paper_2506_02741_b200.mapping import BatchedMapper
    cfg = cached_config(2)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    kf = cfg.keyframes[2]
    m = BatchedMapper(R, pr, co, cfg.intr, [vt.pose_tensor(np.asarray(kf.pose, dtype=np.float32), "cuda")],
                      [dict(rgb=torch.from_numpy(kf.rgb).cuda(), depth=torch.from_numpy(kf.depth).cuda())], 0.8, 1.0)
    m.step(allreduce=False)
    torch.cuda.synchronize()
    eager = [t.clone() for t in m.out] + [m.loss.clone(), m.grads.flat.clone()]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        m.step(allreduce=False)
    m.grads.flat.fill_(123.0)
    for t in m.out:
        t.fill_(-1.0)
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager[:4], list(m.out) + [m.loss]):
        assert torch.equal(a, b)
    assert torch.allclose(eager[4], m.grads.flat, rtol=1e-5, atol=1e-6)


def test_step_host_matches_device_path(vt):
    cfg = cached_config(2)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    tg = cfg.targets[0]
    H, W = cfg.intr.height, cfg.intr.width
    out = tuple(torch.empty(s, device="cuda") for s in ((H, W, 3), (H, W), (H, W)))
    d1 = torch.zeros((cfg.n_slots, 4), device="cuda")
    r1 = torch.zeros(cfg.n_slots, device="cuda")
    loss_h = R.step_host(pr, co, torch.from_numpy(view32(cfg.views[0]).astype(np.float32)), cfg.intr,
                         torch.from_numpy(tg.rgb).pin_memory(), torch.from_numpy(tg.depth).pin_memory(),
                         0.8, 1.0, 0, 0, 0, vt.VTGS_GRAD_ATTR, (0, cfg.n_slots), out, d1, r1)
    v, _ = _render_gpu(vt, R, cfg, pr, co)
    d2 = torch.zeros_like(d1)
    r2 = torch.zeros_like(r1)
    lo = torch.zeros(1, device="cuda")
    R.render_bwd(vt.VTGS_GRAD_ATTR, d_col_opa=d2, d_radius=r2,
                 loss=dict(target_rgb=torch.from_numpy(tg.rgb).cuda(), target_depth=torch.from_numpy(tg.depth).cuda(),
                           w_color=0.8, w_depth=1.0), loss_out=lo)
    torch.cuda.synchronize()
    assert loss_h == pytest.approx(lo.item(), rel=1e-6)
    assert torch.allclose(d1, d2, rtol=1e-5, atol=1e-6)
    # repeated calls with all-pinned host buffers (the way the bench's e2e leg calls it)
    hv = torch.from_numpy(view32(cfg.views[0]).astype(np.float32)).pin_memory()
    hr, hd = torch.from_numpy(tg.rgb).pin_memory(), torch.from_numpy(tg.depth).pin_memory()
    for _ in range(3):
        d3 = torch.zeros_like(d1)
        r3 = torch.zeros_like(r1)
        loss_g = R.step_host(pr, co, hv, cfg.intr, hr, hd, 0.8, 1.0, 0, 0, 0, vt.VTGS_GRAD_ATTR, (0, cfg.n_slots),
                             out, d3, r3)
        assert loss_g == loss_h
        assert torch.allclose(d3, d2, rtol=1e-5, atol=1e-6)
        assert torch.allclose(r3, r2, rtol=1e-5, atol=1e-6)


def test_batched_mapper_deterministic_merge(vt):
    """BatchedMapper(deterministic=True) — the bench's `--deterministic` step — over five views:
    two steps give bit-identical 5N gradient buffers (int64 fixed-point merge), equal to the
    float-atomic step within the summation-order bound of the test above."""
    from paper_2506_02741_b200.mapping import BatchedMapper
    from synth.scenes import perturb_pose
    cfg = cached_config(1)
    R0 = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R0, cfg)
    rng = np.random.default_rng(4)
    views = [vt.pose_tensor(np.asarray(perturb_pose(cfg.keyframes[0].pose, 1.0 * k, 0.01 * k, rng),
                                       dtype=np.float32), "cuda") for k in range(5)]
    tg = cfg.targets[0]
    tgts = [dict(rgb=torch.from_numpy(tg.rgb).cuda(), depth=torch.from_numpy(tg.depth).cuda()) for _ in views]
    det = BatchedMapper(R0, pr, co, cfg.intr, views, tgts, 0.8, 1.0, deterministic=True)
    a = det.step(allreduce=False).flat.clone()
    b = det.step(allreduce=False).flat.clone()
    flt = BatchedMapper(R0, pr, co, cfg.intr, views, tgts, 0.8, 1.0).step(allreduce=False).flat.clone()
    torch.cuda.synchronize()
    assert a.abs().sum() > 0 and torch.equal(a, b)
    assert float((a - flt).norm()) <= 1e-5 * float(flt.norm())


def test_batched_mapper_two_contexts_equals_one(vt):
    """BatchedMapper with its views alternating over two renderer contexts / CUDA streams (the
    bench's configs 4 / 5) gives the same 5N gradient sum and per-view losses as one context: the
    losses exactly (fixed-order reductions), the gradients up to the float-atomic summation order,
    bounded by the per-view gradients' magnitudes."""
    from paper_2506_02741_b200.mapping import BatchedMapper
    from synth.scenes import perturb_pose
    cfg = cached_config(1)
    R0 = _renderer(vt, cfg)
    R1 = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R0, cfg)
    rng = np.random.default_rng(3)
    views = [vt.pose_tensor(np.asarray(perturb_pose(cfg.keyframes[0].pose, 1.0 * k, 0.01 * k, rng),
                                       dtype=np.float32), "cuda") for k in range(5)]
    tg = cfg.targets[0]
    tgts = [dict(rgb=torch.from_numpy(tg.rgb).cuda(), depth=torch.from_numpy(tg.depth).cuda()) for _ in views]
    one = BatchedMapper(R0, pr, co, cfg.intr, views, tgts, 0.8, 1.0)
    two = BatchedMapper([R0, R1], pr, co, cfg.intr, views, tgts, 0.8, 1.0)
    g1 = one.step(allreduce=False).flat.clone()
    l1 = one.loss.clone()
    g2 = two.step(allreduce=False).flat.clone()
    torch.cuda.synchronize()
    assert torch.equal(l1, two.loss)
    scale = torch.zeros_like(g1)
    for i in range(len(views)):   # Σ over views of |that view's gradient|
        single = BatchedMapper(R0, pr, co, cfg.intr, views[i:i + 1], tgts[i:i + 1], 0.8, 1.0)
        scale += single.step(allreduce=False).flat.abs()
    torch.cuda.synchronize()
    assert g1.abs().sum() > 0
    # a lost or doubled view would miss by ~|g_v|; summation order moves single elements by far
    # less than 1e-3 of the per-view magnitudes, and the buffer as a whole by < 1e-5
    assert torch.all((g2 - g1).abs() <= 1e-3 * scale + 1e-6), float((g2 - g1).abs().max())
    assert float((g2 - g1).norm()) <= 1e-5 * float(g1.norm())


def test_step_host_sensor_equals_float_targets(vt):
    """vtgs_step_host_sensor (uint8 RGB + uint16 depth uploaded, widened on the device) is the same
    step as vtgs_step_host on the fp32 targets a host-side conversion with the same two IEEE
    operations gives (c = v / 255, z = d · scale): identical loss and, with the deterministic merge,
    bit-identical gradients; invalid arguments are refused."""
    cfg = cached_config(2)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    tg = cfg.targets[0]
    H, W = cfg.intr.height, cfg.intr.width
    scale = np.float32(1.0 / 5000.0)
    rgb8 = np.clip(np.rint(tg.rgb * 255.0), 0, 255).astype(np.uint8)
    d16 = np.clip(np.rint(tg.depth / scale), 0, 65535).astype(np.uint16)
    rgb_f = rgb8.astype(np.float32) / np.float32(255.0)
    dep_f = d16.astype(np.float32) * scale
    out = tuple(torch.empty(sh, device="cuda") for sh in ((H, W, 3), (H, W), (H, W)))
    hv = torch.from_numpy(view32(cfg.views[0]).astype(np.float32)).pin_memory()
    want = vt.VTGS_GRAD_ATTR | vt.VTGS_GRAD_DETERMINISTIC
    res = []
    for sensor in (False, True):
        d = torch.zeros((cfg.n_slots, 4), device="cuda")
        r = torch.zeros(cfg.n_slots, device="cuda")
        if sensor:
            loss = R.step_host_sensor(pr, co, hv, cfg.intr, torch.from_numpy(rgb8).pin_memory(),
                                      torch.from_numpy(d16).pin_memory(), float(scale), 0.8, 1.0, 0, 0, 0, want,
                                      (0, cfg.n_slots), out, d, r)
        else:
            loss = R.step_host(pr, co, hv, cfg.intr, torch.from_numpy(rgb_f).pin_memory(),
                               torch.from_numpy(dep_f).pin_memory(), 0.8, 1.0, 0, 0, 0, want, (0, cfg.n_slots),
                               out, d, r)
        torch.cuda.synchronize()
        res.append((loss, d.cpu(), r.cpu()))
    assert res[0][0] == res[1][0]
    assert torch.equal(res[0][1], res[1][1]) and torch.equal(res[0][2], res[1][2])
    assert res[0][1].abs().sum() > 0
    with pytest.raises(vt.VtgsError):
        R.step_host_sensor(pr, co, hv, cfg.intr, torch.from_numpy(rgb8), torch.from_numpy(d16), 0.0, 0.8, 1.0,
                           0, 0, 0, want, (0, cfg.n_slots), out, d, r)
    with pytest.raises(vt.VtgsError):   # fp32 depth where uint16 is expected
        R.step_host_sensor(pr, co, hv, cfg.intr, torch.from_numpy(rgb8), torch.from_numpy(dep_f), float(scale),
                           0.8, 1.0, 0, 0, 0, want, (0, cfg.n_slots), out, d, r)


# ------------------------------------------------------------------------------ f1 (head-frame BA)
def _ba_scene(seed=0, W=64, H=48, K=3):
    """K keyframes of a noisy slanted surface 1.5–3 m away, a view between keyframes 0 and 1."""
    from synth.scenes import perturb_pose
    rng = np.random.default_rng(seed)
    intr = Intrinsics(60.0, 60.0, (W - 1) / 2, (H - 1) / 2, W, H)
    base = np.array([1.0, 0, 0, 0, 0, 0, 0])
    poses = np.stack([perturb_pose(base, 2.0 * k, 0.03 * k, rng) for k in range(K)]).astype(np.float32)
    xs, ys = np.meshgrid(np.arange(W), np.arange(H))
    depth = np.stack([1.5 + 1.5 * xs / W + 0.3 * ys / H + rng.normal(0, 0.01, (H, W)) for _ in range(K)])
    depth[:, rng.random((H, W)) < 0.01] = 0.0
    rgb = rng.uniform(0, 1, (K, H, W, 3))
    opa = 1 / (1 + np.exp(-rng.normal(size=(K, H, W))))
    view = perturb_pose(poses[0].astype(np.float64), 1.0, 0.015, rng)
    return intr, poses, depth.astype(np.float32), rgb.astype(np.float32), opa.astype(np.float32), view


@pytest.mark.parametrize("scene", ["ba_small", "config2"])
def test_position_and_keyframe_pose_gradient_parity(vt, scene):
    """Head-frame bundle adjustment: dL/dX_w per Gaussian (VTGS_GRAD_POSITION)
    within the gradient bar (1e-3 rel / 1e-5 abs, or the fp32 summation floor, R23, or
    a T cut-off near-tie's allowance) on Gaussians not tainted by an α near-tie, and the
    per-keyframe pose gradients (vtgs_keyframe_pose_grad) within 1e-3 of their norm, against the
    oracle's or_render_bwd d_pos + or_keyframe_pose_grad — on a small 3-keyframe scene and on
    config 2 at full size (5 keyframes, 1200×680, 4.08M slots, the view = keyframe 2's pose)."""
    if scene == "ba_small":
        intr, poses, depth, rgb, opa, view = _ba_scene()
    else:
        cfg = cached_config(2)
        intr, poses, depth, rgb, opa = cfg.intr, cfg.pose_stack(), cfg.depth_stack(), cfg.rgb_stack(), cfg.opacity
        view = cfg.views[0]
    K, H, W = depth.shape
    N = K * H * W
    R = vt.Renderer(0, N, W, H)
    dev = "cuda"
    pr, co = R.instantiate(torch.from_numpy(depth).to(dev), torch.from_numpy(rgb).to(dev),
                           vt.pose_tensor(poses, dev), intr, torch.from_numpy(opa).to(dev))
    v = vt.pose_tensor(view32(view), dev)
    out = R.render_fwd(pr, co, v, intr)
    rng = np.random.default_rng(3)
    gC = rng.normal(size=(H, W, 3)).astype(np.float32)
    gD = rng.normal(size=(H, W)).astype(np.float32)
    gS = rng.normal(size=(H, W)).astype(np.float32)
    dpos = torch.zeros((N, 4), device=dev)
    dpose = torch.zeros(7, device=dev)
    R.render_bwd(vt.VTGS_GRAD_POSITION | vt.VTGS_GRAD_POSE, d_position=dpos, d_pose=dpose,
                 dL_dcolor=torch.from_numpy(gC).to(dev), dL_ddepth=torch.from_numpy(gD).to(dev),
                 dL_dsil=torch.from_numpy(gS).to(dev))
    kf_gpu = R.keyframe_pose_grad(pr, dpos, vt.pose_tensor(poses, dev), H * W).cpu().numpy().astype(np.float64)
    torch.cuda.synchronize()
    del out
    opr, oco, _ = oracle.instantiate(depth, rgb, poses.astype(np.float64), intr, opa)
    ref = oracle.render(opr, oco, view32(view), intr, want_tainted=True)
    g = oracle.render_bwd(opr, oco, view32(view), intr, gC, gD, gS, want_allow=True)
    keep = ~ref["tainted"]
    d = dpos.cpu().numpy()[:, :3].astype(np.float64)
    st = {}
    dk, rk = d[keep], g["d_pos"][keep]
    ok = close(dk, rk, absum=g["d_pos_abs"][keep], stats=st)
    a_ok = np.abs(dk - rk) <= g["d_allow"][keep, 5:8] + np.maximum(1e-5, 1e-3 * np.abs(rk))
    n_allow = int((a_ok & ~ok).any(1).sum())
    ok |= a_ok
    assert ok.all(), report("d_position", ok, dk, rk)
    assert st["floor_only"] <= 5 + 1e-5 * st["n"], st
    touched = g["d_pos_abs"].sum(1) > 0
    frac = (int((~keep & touched).sum()) + n_allow) / max(int(touched.sum()), 1)
    print(f"[parity BA {scene}] tainted {int((~keep & touched).sum())}, allowance-only {n_allow}, "
          f"excluded fraction {frac:.2e}")
    assert frac <= 5e-3
    assert np.linalg.norm(dpose.cpu().numpy() - g["d_pose"]) <= 1e-3 * np.linalg.norm(g["d_pose"])
    kf_ref = oracle.keyframe_pose_grad(depth, poses.astype(np.float64), intr, g["d_pos"])
    for k in range(K):
        assert np.linalg.norm(kf_gpu[k] - kf_ref[k]) <= 1e-3 * np.linalg.norm(kf_ref[k]), (k, kf_gpu[k], kf_ref[k])


def test_view_tied_pose_invariance_gpu(vt):
    """A keyframe rendered from its own pose: view-pose and owner-pose gradients cancel
    (d_pose + d_kf_pose = 0 up to fp32 summation, PAPER.md:119 view-tied centres)."""
    intr, poses, depth, rgb, opa, _ = _ba_scene(seed=1, K=1)
    K, H, W = depth.shape
    N = K * H * W
    R = vt.Renderer(0, N, W, H)
    dev = "cuda"
    pt = vt.pose_tensor(poses, dev)
    pr, co = R.instantiate(torch.from_numpy(depth).to(dev), torch.from_numpy(rgb).to(dev), pt, intr,
                           torch.from_numpy(opa).to(dev))
    out = R.render_fwd(pr, co, pt[0:1].clone(), intr)
    rng = np.random.default_rng(5)
    dpos = torch.zeros((N, 4), device=dev)
    dpose = torch.zeros(7, device=dev)
    R.render_bwd(vt.VTGS_GRAD_POSITION | vt.VTGS_GRAD_POSE, d_position=dpos, d_pose=dpose,
                 dL_dcolor=torch.from_numpy(rng.normal(size=(H, W, 3)).astype(np.float32)).to(dev))
    kf = R.keyframe_pose_grad(pr, dpos, pt, H * W)[0]
    torch.cuda.synchronize()
    del out
    s = dpose.abs().max().item()
    assert s > 1e-2
    assert (dpose + kf).abs().max().item() <= 2e-3 * s, (dpose.cpu().numpy(), kf.cpu().numpy())


# ------------------------------------------------------------------------------ f2 (SSIM of Eq. 2)
@pytest.mark.parametrize("size", [(64, 48), (37, 29), (11, 11), (200, 50), (1200, 680)])
def test_ssim_loss_parity(vt, size):
    """τ·L_S of Eq. 2 (R24) and its gradient against the oracle's plain
    121-tap window definition: loss within 1e-5 relative; gradient within 1e-3 relative or 1e-5
    absolute (the north_star gradient bar) elementwise, including the ragged borders, the halos
    between CTA columns / rows (200×50: 4 tile columns; 1200×680: the mapping view)."""
    W, H = size
    rng = np.random.default_rng(W * H)
    x = rng.uniform(size=(H, W, 3)).astype(np.float32)
    y = np.clip(x + rng.normal(0, 0.1, size=x.shape), 0, 1).astype(np.float32)
    R = vt.Renderer(0, 16, W, H)
    d = torch.zeros((H, W, 3), device="cuda")
    loss = torch.zeros(1, device="cuda")
    R.ssim_loss(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), 0.2, d_color=d, loss_out=loss)
    torch.cuda.synchronize()
    ref_loss, ref_g = oracle.ssim_loss(x, y, 0.2)
    assert abs(loss.item() - ref_loss) <= 1e-5 * abs(ref_loss)
    g = d.cpu().numpy().astype(np.float64)
    ok = close(g, ref_g)
    assert ok.all(), report("ssim grad", ok, g, ref_g)


def test_ssim_errors_and_accumulate(vt):
    R = vt.Renderer(0, 16, 64, 48)
    x = torch.rand((10, 12, 3), device="cuda")
    with pytest.raises(vt.VtgsError):
        R.ssim_loss(x, x)                       # smaller than the 11×11 window
    x = torch.rand((48, 64, 3), device="cuda")
    y = torch.rand((48, 64, 3), device="cuda")
    d1 = torch.zeros_like(x)
    R.ssim_loss(x, y, 0.2, d_color=d1)
    d2 = d1.clone()
    R.ssim_loss(x, y, 0.2, d_color=d2)          # accumulates
    torch.cuda.synchronize()
    assert torch.allclose(d2, 2 * d1, rtol=1e-6, atol=0)


def test_mapping_objective_with_ssim_parity(vt):
    """The full mapping objective of Eq. 2, ρ‖V − V'‖₁ + τ L_S + σ U‖D − D'‖₁ (ρ, τ, σ = 0.8, 0.2,
    1.0), on config 1: SSIM gradient from vtgs_ssim_loss passed as the fused loss's
    extra colour upstream; colour / opacity / radius gradients against the oracle."""
    cfg = cached_config(1)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    _, out = _render_gpu(vt, R, cfg, pr, co)
    tg = cfg.targets[0]
    H, W = cfg.intr.height, cfg.intr.width
    trgb = torch.from_numpy(tg.rgb).cuda()
    dss = torch.zeros((H, W, 3), device="cuda")
    R.ssim_loss(out[0], trgb, 0.2, d_color=dss)
    L = dict(target_rgb=trgb, target_depth=torch.from_numpy(tg.depth).cuda(), w_color=0.8, w_depth=1.0,
             extra_dcolor=dss)
    want = vt.VTGS_GRAD_ATTR
    dco, drad, dpose = _run_bwd(vt, R, cfg, want, cfg.n_slots, loss=L)
    opr, oco = oracle_instantiate(cfg)
    v = _view(cfg)
    img = oracle.render(opr, oco, v, cfg.intr)
    _, gC, gD, gS, lflags, flip = oracle.l1_upstream(img["color"], img["depth"], img["sil"], tg.rgb, tg.depth,
                                                     None, 0.8, 1.0, 0, 0, 0, want_flip=True)
    _, gss = oracle.ssim_loss(img["color"], tg.rgb, 0.2)
    ref, g, allow = _oracle_grads(cfg, opr, oco, v, gC + gss, gD, gS, flip=flip)
    _check_grads(want, dco, drad, dpose, g, ref["tainted"], vt, allow=allow, name="mapping objective + SSIM")


# ------------------------------------------------------------------------------ f4 (densification)
def test_densify_parity(vt):
    """Regular-frame densification: on a synthetic silhouette field given to
    both sides, the appended Gaussians are bit-exact with the oracle (same rows, same order,
    same count), including a pixel exactly at the threshold and invalid depths."""
    rng = np.random.default_rng(11)
    H, W = 37, 53
    intr = Intrinsics(40.0, 41.0, (W - 1) / 2, (H - 1) / 2, W, H)
    depth = np.where(rng.random((H, W)) < 0.1, 0.0, rng.uniform(0.5, 4.0, (H, W))).astype(np.float32)
    rgb = rng.random((H, W, 3)).astype(np.float32)
    sil = rng.random((H, W)).astype(np.float32)
    sil[3, 4] = 0.5
    depth[3, 4] = 2.0
    opa = rng.random((H, W)).astype(np.float32)
    from synth.scenes import perturb_pose
    pose = perturb_pose(np.array([1.0, 0, 0, 0, 0, 0, 0]), 7.0, 0.3, rng).astype(np.float32)
    R = vt.Renderer(0, H * W, W, H)
    dev = "cuda"
    out_pr = torch.zeros((H * W, 4), device=dev)
    out_co = torch.zeros((H * W, 4), device=dev)
    n = R.densify(torch.from_numpy(depth).to(dev), torch.from_numpy(rgb).to(dev), vt.pose_tensor(pose, dev), intr,
                  torch.from_numpy(sil).to(dev), out_pr, out_co, 0.5, torch.from_numpy(opa).to(dev))
    opr, oco = oracle.densify(depth, rgb, pose.astype(np.float64), intr, sil, 0.5, opa)
    assert n == len(opr)
    assert np.array_equal(out_pr.cpu().numpy()[:n], opr.astype(np.float32))
    assert np.array_equal(out_co.cpu().numpy()[:n], oco.astype(np.float32))
    assert not out_pr.cpu().numpy()[n:].any()


def test_densify_after_render(vt):
    """End to end: render the section (config 3's keyframes) from the frame to track, densify
    where the rendered silhouette is < 0.5; the new set equals the oracle's {valid ∧ S < 0.5}
    except at pixels whose silhouette lies within 1e-4 of the threshold (the render bar)."""
    cfg = cached_config(3)
    R = _renderer(vt, cfg)
    pr, co = gpu_instantiate(R, cfg)
    v = view32(cfg.extra["gt_pose"])
    vv, out = _render_gpu(vt, R, cfg, pr, co, v)
    tg = cfg.targets[0]
    H, W = cfg.intr.height, cfg.intr.width
    dev = "cuda"
    out_pr = torch.zeros((H * W, 4), device=dev)
    out_co = torch.zeros((H * W, 4), device=dev)
    n = R.densify(torch.from_numpy(tg.depth).to(dev), torch.from_numpy(tg.rgb).to(dev), vv, cfg.intr, out[2],
                  out_pr, out_co, 0.5)
    opr, oco = oracle_instantiate(cfg)
    img = oracle.render(opr, oco, v, cfg.intr)
    near = np.abs(img["sil"] - 0.5) <= 1e-4
    sel = (tg.depth > 0) & (img["sil"] < 0.5)
    assert abs(n - int(sel.sum())) <= int(near.sum())
    # the oracle's densification of its own silhouette, compared on pixels away from the threshold
    dpr, _ = oracle.densify(tg.depth, tg.rgb, v, cfg.intr, img["sil"], 0.5)
    g = out_pr.cpu().numpy()[:n]
    if not near.any():
        assert np.array_equal(g, dpr.astype(np.float32))


# ------------------------------------------------------------------------------ f3 (visibility, pre-tracking)
def test_visibility_mask_parity(vt):
    """the frame to track (config 3) against its section's head, middle and last
    keyframes — bit-exact with the oracle's fp32 decisions (same operation order, R25)."""
    cfg = cached_config(3)
    R = _renderer(vt, cfg)
    tg = cfg.targets[0]
    K = cfg.K
    idx = [0, K // 2, K - 1]
    kd = cfg.depth_stack()[idx]
    kp = cfg.pose_stack()[idx].astype(np.float32)
    pose = view32(cfg.views[0]).astype(np.float32)
    m = R.visibility_mask(torch.from_numpy(tg.depth).cuda(), vt.pose_tensor(pose, "cuda"),
                          torch.from_numpy(np.ascontiguousarray(kd)).cuda(), vt.pose_tensor(kp, "cuda"), cfg.intr)
    ref = oracle.visibility(tg.depth, pose.astype(np.float64), kd, kp.astype(np.float64), cfg.intr)
    g = m.cpu().numpy().astype(bool)
    assert 0.05 < ref.mean() < 1.0
    assert np.array_equal(g, ref), int((g != ref).sum())


def test_pretrack_select_concurrent_matches_sequential(vt):
    """PAPER.md:180-182 pre-tracking: three candidate sections (config 3's keyframes split in
    three) tracked for 10 iterations each, concurrently on three streams; the losses equal a
    sequential run bit for bit, the selection is their argmin, and the selected section's
    pre-tracking reduces its rendering error."""
    from paper_2506_02741_b200 import tracking
    cfg = cached_config(3)
    tg = cfg.targets[0]
    dev = "cuda"
    rgb, depth = torch.from_numpy(tg.rgb).to(dev), torch.from_numpy(tg.depth).to(dev)
    init = vt.pose_tensor(view32(cfg.views[0]), dev)
    H, W = cfg.intr.height, cfg.intr.width
    groups = [[0, 1, 2], [3, 4, 5], [6, 7, 8, 9]]
    secs, rends = [], []
    for gidx in groups:
        n = len(gidx) * H * W
        Rg = vt.Renderer(0, n, W, H)
        ds = torch.from_numpy(np.ascontiguousarray(cfg.depth_stack()[gidx])).to(dev)
        ps = vt.pose_tensor(cfg.pose_stack()[gidx], dev)
        pr, co = Rg.instantiate(ds, torch.from_numpy(np.ascontiguousarray(cfg.rgb_stack()[gidx])).to(dev), ps,
                                cfg.intr, torch.from_numpy(np.ascontiguousarray(cfg.opacity[gidx])).to(dev))
        vis = tracking.section_visibility(Rg, depth, init, ds, ps, cfg.intr)
        secs.append(dict(pos_rad=pr, col_opa=co, vis_mask=vis))
        rends.append(Rg)
    best, finals, res = tracking.pretrack_select(rends, secs, cfg.intr, rgb, depth, init, 10, 0.002, 0.002)
    best2, finals2, _ = tracking.pretrack_select(rends, secs, cfg.intr, rgb, depth, init, 10, 0.002, 0.002,
                                                 concurrent=False)
    assert finals == finals2 and best == best2 == int(np.argmin(finals))
    ls = res[best].losses.cpu().numpy()
    assert ls[-1] < ls[0]                      # the selected section's pre-tracking reduces the error


# ------------------------------------------------------------------------------ f3 (head-frame selection)
def test_select_overlap_section_matches_oracle(vt):
    """The whole head-frame selection of PAPER.md:180-182 / SPEC.md:382-390 against an independent
    oracle recomputation: per-candidate visible-point counts (vtgs_visibility_counts) bit-exact
    with the oracle's, the same γ-filtered most-front sections, per-section visibility masks
    bit-exact, the pre-track final Eq. 1 losses of each section within 2e-3 relative of the
    oracle's own tracking loop (its own renders, Adam steps and masks), and the same argmin
    ("chosen section = argmin of independently recomputed pre-track losses")."""
    from paper_2506_02741_b200 import tracking
    from synth.scenes import pretrack_scene
    sc = pretrack_scene(0)
    intr = sc["intr"]
    H, W = intr.height, intr.width
    dev = "cuda"
    frames = sc["frames"]
    head = sc["head"]
    cand = sc["candidates"]
    cand_depth = np.stack([frames[i].depth for i in cand])
    cand_poses = np.stack([frames[i].pose for i in cand]).astype(np.float32)
    init = view32(sc["init"])
    renderers = [vt.Renderer(0, 2 * H * W, W, H) for _ in range(3)]
    sections_gpu, sections_or = [], []
    hd, hr = torch.from_numpy(head.depth).to(dev), torch.from_numpy(head.rgb).to(dev)
    init_t = vt.pose_tensor(init, dev)
    for sec in sc["sections"]:
        fr = sec["frames"]
        depth = np.stack([frames[i].depth for i in fr])
        rgb = np.stack([frames[i].rgb for i in fr])
        poses = np.stack([frames[i].pose for i in fr]).astype(np.float32)
        opa = sc["opacity"][fr]
        pr, co = renderers[0].instantiate(torch.from_numpy(depth).to(dev), torch.from_numpy(rgb).to(dev),
                                          vt.pose_tensor(poses, dev), intr, torch.from_numpy(opa).to(dev))
        vf = sec["vis_frames"]
        vdepth = np.stack([frames[i].depth for i in vf])
        vposes = np.stack([frames[i].pose for i in vf]).astype(np.float32)
        vis = tracking.section_visibility(renderers[0], hd, init_t, torch.from_numpy(vdepth).to(dev),
                                          vt.pose_tensor(vposes, dev), intr)
        sections_gpu.append({"pos_rad": pr.clone(), "col_opa": co.clone(), "vis_mask": vis.clone()})
        opr, oco, _ = oracle.instantiate(depth, rgb, poses.astype(np.float64), intr, opa)
        ovis = oracle.visibility(head.depth, init, vdepth, vposes.astype(np.float64), intr)
        assert np.array_equal(vis.cpu().numpy().astype(bool), ovis)
        sections_or.append((opr, oco, ovis))
    torch.cuda.synchronize()
    chosen, secs, finals, counts, nv = tracking.select_overlap_section(
        renderers, sections_gpu, hd, hr, init_t, torch.from_numpy(cand_depth).to(dev),
        vt.pose_tensor(cand_poses, dev), sc["cand_section"], intr, sc["gamma"], sc["iterations"], sc["lr"], sc["lr"])
    ocounts, onv = oracle.visibility_counts(head.depth, init, cand_depth, cand_poses.astype(np.float64), intr)
    assert counts == ocounts and nv == onv, (counts, ocounts, nv, onv)
    osecs = oracle.select_sections(ocounts, onv, sc["cand_section"], sc["gamma"])
    assert secs == osecs, (secs, osecs)
    assert len(secs) >= 2, f"the scene should offer a choice: {secs} from counts {counts} / {nv}"
    ofinals = []
    for k in osecs:
        opr, oco, ovis = sections_or[k]
        _, losses = oracle.track(opr, oco, intr, head.rgb, head.depth, init, sc["iterations"], sc["lr"], sc["lr"],
                                 vis=ovis)
        ofinals.append(losses[-1])
    for a, b in zip(finals, ofinals):
        assert abs(a - b) <= 2e-3 * abs(b), (finals, ofinals)
    ob = int(np.argmin(ofinals))
    srt = sorted(ofinals)
    assert srt[1] - srt[0] > 1e-2 * srt[0], f"near-tie in the oracle's losses {ofinals}"
    assert chosen == osecs[ob], (chosen, osecs, finals, ofinals)
    print(f"[f3] counts {counts} / {nv}; sections {secs}; final losses gpu {finals} oracle {ofinals}; chosen {chosen}")

"""The oracle against the small worked examples the paper and SPEC print, kept as cited text
fixtures under tests/golden/ (task rule ③).  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle
from synth.scenes import Intrinsics

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        d = json.load(f)
    assert d.get("cite"), f"{name} must cite its source"
    return d


@pytest.mark.parametrize("mode", ["f32", "f64"])
def test_golden_back_project(mode):
    g = _load("spec_back_project.json")
    i = g["intrinsics"]
    intr = Intrinsics(i["fx"], i["fy"], i["cx"], i["cy"], i["width"], i["height"])
    for case in g["cases"]:
        depth = np.zeros((1, i["height"], i["width"]))
        x, y = case["pixel"]
        depth[0, y, x] = case["depth"]
        pr, _, n = oracle.instantiate(depth, np.zeros((1, i["height"], i["width"], 3)), np.array([case["pose"]]),
                                      intr, mode=mode)
        assert n == 1, case["cite"]
        np.testing.assert_array_equal(pr[y * i["width"] + x, :3], case["world"], err_msg=case["cite"])


def test_golden_radius_and_footprint():
    g = _load("paper_radius_footprint.json")
    for c in g["cases"]:
        W = H = 8
        intr = Intrinsics(c["f"], c["f"], 3.5, 3.5, W, H)
        depth = np.zeros((1, H, W))
        depth[0, 3, 3] = c["depth"]
        pr, _, _ = oracle.instantiate(depth, np.zeros((1, H, W, 3)), np.array([[1.0, 0, 0, 0, 0, 0, 0]]), intr,
                                      mode="f64")
        assert abs(pr[3 * W + 3, 3] - c["radius"]) < 1e-15
        # render it from a camera z_view in front: sigma = f r / z
        view = np.array([1.0, 0, 0, 0, 0, 0, c["depth"] - c["z_view"]])
        p = oracle.project(pr, view, intr, mode="f64")
        assert abs(p["proj"][3 * W + 3, 3] - c["sigma_px"]) < 1e-12


def test_golden_l1_example():
    """α = 0.5, β = 0.025 with unit colour error and zero depth error, full mask
    (mean form) → 0.5."""
    g = _load("paper_hyperparameters.json")["l1_example"]
    H, W = 4, 5
    C = np.ones((H, W, 3)) * 0.75
    tC = C - g["color_error"] / 3.0            # ‖·‖₁ over 3 channels = 1 per pixel
    D = np.full((H, W), 2.0)
    S = np.ones((H, W))
    loss, *_ = oracle.l1_upstream(C, D, S, tC, D.copy(), None, g["alpha"], g["beta"], 1, 1, 1)
    assert abs(loss - g["loss"]) < 1e-12


def test_golden_hyperparameters_are_the_configs():
    """The bench / mapping driver use the paper's mapping weights."""
    from synth.scenes import cached_config
    g = _load("paper_hyperparameters.json")
    wc, wd = cached_config(2).loss_weights
    assert (wc, wd) == (g["mapping"]["rho"], g["mapping"]["sigma"])


def test_golden_ssim_constant_images():
    g = _load("spec_ssim_constant.json")
    H, W = 14, 15
    for c in g["cases"]:
        _, _, smap = oracle.ssim_loss(np.full((H, W, 3), c["a"]), np.full((H, W, 3), c["b"]), want_map=True)
        np.testing.assert_allclose(smap[5:H - 5, 5:W - 5], c["ssim_interior"], rtol=1e-12, atol=0)

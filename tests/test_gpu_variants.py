"""The A/B kernel variants (VTGS_FWD, VTGS_BWD_*, VTGS_SORT — read once per
process) each keep parity: a subprocess per variant runs the smoke check (config 1 instantiate,
bit-exact tile lists, forward images and all gradients against the oracle) and the long-list sort
paths.  A variant that silently broke (the radix-only sort once sorted only tile 0) fails here.
VTGS_LIB=checked runs the same checks on the bounds-checked build (libvtgs_checked.so: in-kernel
index / invariant checks that trap) — compute-sanitizer is closed on this GPU pool."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("var", ["VTGS_SORT=0", "VTGS_FWD=8", "VTGS_FWD=4", "VTGS_FWD=14", "VTGS_BWD_POSE=0", "VTGS_BWD_MINB=12",
                                 "VTGS_BWD_RING=1", "VTGS_LIB=checked"])
def test_variant_parity(var):
    k, v = var.split("=")
    env = dict(os.environ, **{k: v})
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "smoke ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-q", "-m", "gpu", "-x",
                        "-k", "sort_paths or micro_ragged or pose_only_upstream"
                        + (" or fused_l1 or long_lists or tracking_loop or densify or visibility or ssim_loss_parity"
                           if var == "VTGS_LIB=checked" else "")
                        + (" or fused_l1 or upstream or deterministic or long_lists" if var == "VTGS_BWD_RING=1" else "")],
                       cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]

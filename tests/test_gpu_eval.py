"""evaluate_map_quality on the device (vrf_evaluate_views: views rendered and
scored in HBM) against the reference's own evaluate_map_quality
(eval.cpp:210-240, oracle/_ref) on the same grid and frames.

Sample counts are exact (the rendered-depth mask is a hit decision, bit-exact
with the reference); PSNR and depth L1 agree to 1e-9 relative (renders agree
to ~1e-12; the device sums in a fixed block order, the reference sequentially).
"""
import numpy as np
import pytest

from paper_2307_03404_b200 import metrics
from paper_2307_03404_b200.api import RenderParams

from scenes import fresh_grid, room_scene

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("which", ["gt", "fresh"])
@pytest.mark.parametrize("seed", [0, 3])
def test_evaluate_map_quality_matches_reference(ctx, ref, which, seed):
    grid, intr, frames = room_scene(res=33, width=64, height=48, n_frames=3)
    g = grid if which == "gt" else fresh_grid(grid, sigma_init=2.0, seed=seed)
    ctx.load_grid(g)
    idx = [0, 2, 1]
    q = metrics.evaluate_map_quality(ctx, intr, frames, idx, images=6, pixels_per_image=500,
                                     seed=seed)
    gh, fh = ref.grid(g), ref.frames(frames, intr)
    try:
        p, l1, ns, npx = ref.evaluate_map_quality(gh, fh, intr, idx, RenderParams(), images=6,
                                                  pixels_per_image=500, seed=seed, threads=1)
    finally:
        ref.lib.ref_grid_destroy(gh)
        ref.lib.ref_frames_destroy(fh)
    assert q.color_samples == ns and q.depth_pixels == npx
    assert q.psnr_db == pytest.approx(p, rel=1e-9)
    assert q.depth_l1_m == pytest.approx(l1, rel=1e-9)


def test_evaluate_map_quality_errors(ctx):
    grid, intr, frames = room_scene()
    ctx.load_grid(grid)
    with pytest.raises(RuntimeError, match="no frames"):
        metrics.evaluate_map_quality(ctx, intr, frames, [])
    empty = fresh_grid(grid)
    empty.set_all_active(False)
    ctx.load_grid(empty)
    with pytest.raises(RuntimeError, match="no valid pixels"):
        metrics.evaluate_map_quality(ctx, intr, frames, [0], images=2, pixels_per_image=20)

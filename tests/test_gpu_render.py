"""Render front-end parity: camera rays, BVH closest hits, dispatch and
surface vertex fields on the GPU against the CPU oracle (brute-force hits), following the
reference's test_geometry.cpp ("bvh agrees with brute force on random soups", "degenerate ray
direction throws", "builtin scenes finalize ...") at equality instead of Approx."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _render():
    from paper_2510_07868_b200 import render
    return render


def _hits_agree(gpu_t, gpu_tri, ref_t, ref_tri):
    """Equal hits; a different triangle is allowed only on an exact t tie (two triangles sharing
    an edge, visited in a different order by the BVH than by the brute-force loop)."""
    gpu_tri = gpu_tri.astype(np.uint32)
    assert np.array_equal(gpu_t.view(np.uint32), ref_t.view(np.uint32))
    diff = gpu_tri != ref_tri
    assert diff.mean() < 0.01, f"{diff.sum()} triangle mismatches"
    return diff


@pytest.mark.parametrize("name", ["cornell", "caustic", "furnace"])
def test_builtin_scene_depth1_matches_oracle(name):
    render = _render()
    desc = getattr(render, f"make_{name}_scene")()
    w, h, seed, frame = 96, 64, 0x5EED, 3
    sc = render.GpuScene(desc)
    g = {k: (v.cpu().numpy() if v is not None else None) for k, v in sc.render_depth1(w, h, seed, frame).items()}
    sc.check()
    ref = oracle.render_depth1(desc, w, h, seed, frame)
    assert np.array_equal(g["o"].view(np.uint32), ref["o"].view(np.uint32))
    assert np.array_equal(g["d"].view(np.uint32), ref["d"].view(np.uint32))
    assert np.array_equal(g["path_key"].view(np.uint64), ref["path_key"])
    diff = _hits_agree(g["t"], g["tri"], ref["t"], ref["tri"])
    same = ~diff
    assert np.array_equal(g["class"][same], ref["class"][same])
    assert np.array_equal(g["p01"][same].view(np.uint32), ref["p01"][same].view(np.uint32))
    assert np.array_equal(g["roughness"][same], ref["roughness"][same])
    # acosf / atan2f: CUDA's and glibc's differ by at most a couple of ulp
    np.testing.assert_allclose(g["wo01"][same], ref["wo01"][same], rtol=0, atol=2e-6)
    surf = g["class"] == render.CLASS_SURFACE
    assert surf.sum() > 0.5 * w * h
    # the center camera ray hits something in a closed scene (test_geometry.cpp:355-363)
    assert g["tri"][(h // 2) * w + w // 2] != -1


@pytest.mark.parametrize("with_tmax", [False, True])
def test_bvh_matches_brute_force_random_soup(with_tmax):
    render = _render()
    pos, idx, mid = oracle.random_soup(500, 5)
    desc = render.SceneDesc(positions=list(pos), indices=list(idx), material_ids=list(mid),
                            materials=[render.Material()])
    sc = render.GpuScene(desc)
    assert sc.node_count > 1
    o, d, tm = oracle.random_rays(10000, 99 if not with_tmax else 100, 1 if not with_tmax else 2,
                                  extent=8.0 if not with_tmax else 6.0, t_max=with_tmax)
    dev = sc.device
    hits = sc.intersect(torch.from_numpy(o).to(dev), torch.from_numpy(d).to(dev),
                        torch.from_numpy(tm).to(dev) if with_tmax else None, check=True)
    ref = oracle.intersect_brute(pos, idx, o, d, tm if with_tmax else None)
    t, tri = hits["t"].cpu().numpy(), hits["tri"].cpu().numpy()
    diff = _hits_agree(t, tri, ref["t"], ref["tri"])
    same = ~diff
    assert np.array_equal(hits["u"].cpu().numpy()[same].view(np.uint32), ref["u"][same].view(np.uint32))
    assert np.array_equal(hits["v"].cpu().numpy()[same].view(np.uint32), ref["v"][same].view(np.uint32))
    assert (tri != -1).sum() > 1000  # the oracle must actually exercise hits


def test_large_mesh_sampled_against_brute_force():
    render = _render()
    pos, idx, mid = oracle.random_soup(20000, 21)
    desc = render.SceneDesc(positions=list(pos), indices=list(idx), material_ids=list(mid),
                            materials=[render.Material()])
    sc = render.GpuScene(desc)
    o, d, _ = oracle.random_rays(1 << 18, 77, 3, extent=6.0)
    dev = sc.device
    hits = sc.intersect(torch.from_numpy(o).to(dev), torch.from_numpy(d).to(dev), check=True)
    t, tri = hits["t"].cpu().numpy(), hits["tri"].cpu().numpy()
    sample = np.arange(0, o.shape[0], 131)
    ref = oracle.intersect_brute(pos, idx, o[sample], d[sample])
    _hits_agree(t[sample], tri[sample], ref["t"], ref["tri"])
    assert (tri != -1).mean() > 0.3


def test_degenerate_direction_raises_and_empty_scene_misses():
    render = _render()
    from paper_2510_07868_b200 import _capi
    pos, idx, mid = oracle.random_soup(10, 3)
    sc = render.GpuScene(render.SceneDesc(positions=list(pos), indices=list(idx), material_ids=list(mid),
                                          materials=[render.Material()]))
    dev = sc.device
    o = torch.zeros(4, 3, device=dev)
    d = torch.tensor([[0, 0, 1], [0, 0, 0], [1, 0, 0], [float("nan"), 0, 1]], dtype=torch.float32, device=dev)
    with pytest.raises(_capi.NrrsError, match="degenerate ray direction"):
        sc.intersect(o, d, check=True)
    sc.check()  # the flag was cleared
    empty = render.GpuScene(render.SceneDesc(materials=[render.Material()]), ctx=sc.ctx)
    assert empty.node_count == 0
    h = empty.intersect(o[:1], d[:1], check=True)
    assert h["tri"].item() == -1 and h["t"].item() == float("inf")


def test_scene_create_rejects_bad_indices():
    render = _render()
    from paper_2510_07868_b200 import _capi
    desc = render.make_cornell_scene()
    desc.indices[5] = 10_000
    with pytest.raises(_capi.NrrsError):
        render.GpuScene(desc)
    desc = render.make_cornell_scene()
    desc.material_ids[0] = 9
    with pytest.raises(_capi.NrrsError):
        render.GpuScene(desc)

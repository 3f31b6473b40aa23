"""GPU: the suffix side of trace_frame against the oracle, bit for bit:
ordered film / parent folds, the reverse pass, TrainSample emission with k_i, Film updates."""
from __future__ import annotations

import json
import pathlib

import numpy as np
import pytest
import torch

import oracle as orc

pytestmark = pytest.mark.gpu
GOLDEN = pathlib.Path(__file__).parent / "golden"


@pytest.fixture(scope="module")
def sx():
    from paper_2510_07868_b200.film import SuffixStage
    s = SuffixStage(0)
    yield s
    s.close()


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_fold_ordered_bitexact(sx):
    g = np.random.default_rng(1)
    n, m = 300001, 40000
    keys = np.concatenate([np.full(17, -1), np.sort(g.integers(0, m, n - 17))]).astype(np.int32)
    terms = g.standard_normal((n, 3)) * np.exp(g.standard_normal((n, 1)) * 4)
    dst = g.standard_normal((m, 3))
    ref = dst.copy()
    orc.fold_ordered(ref, keys, terms)
    d = _cuda(dst)
    sx.fold_ordered(d, _cuda(keys), _cuda(terms))
    np.testing.assert_array_equal(d.cpu().numpy(), ref)


def test_fold_ordered_rejects_out_of_order_and_out_of_range(sx):
    from paper_2510_07868_b200 import _capi
    d = torch.zeros((4, 3), dtype=torch.float64, device="cuda")
    t = torch.ones((3, 3), dtype=torch.float64, device="cuda")
    for keys in ([0, 2, 1], [0, 1, 4]):
        with pytest.raises(_capi.NrrsError) as ei:
            sx.fold_ordered(d, torch.tensor(keys, dtype=torch.int32, device="cuda"), t)
        assert ei.value.code == _capi.NRRS_EINVAL


def test_reverse_pass_emission_k_i_bitexact(sx):
    from paper_2510_07868_b200.film import TRAIN_SAMPLE_DTYPE
    npx = 50000
    verts = orc.gen_vertex_tree([npx, 70001, 52000, 30000], npx)
    i_acc = np.random.default_rng(3).random((npx, 3), dtype=np.float32)
    gv = [None] + [{k: _cuda(a) for k, a in v.items()} for v in verts[1:]]
    sx.reverse_pass(gv)
    orc.reverse_pass(verts)
    for d in range(1, len(verts)):
        np.testing.assert_array_equal(gv[d]["s"].cpu().numpy(), verts[d]["s"], err_msg=f"depth {d}")
    ref, ref_nf = orc.emit_train(verts, i_acc, npx)
    out = torch.zeros((sum(v["pixel"].size for v in verts[1:]), 80), dtype=torch.uint8, device="cuda")
    count, nf = sx.emit_train(gv, _cuda(i_acc), npx, out)
    assert (count, nf) == (len(ref), ref_nf) and nf > 0
    got = out[:count].cpu().numpy().view(TRAIN_SAMPLE_DTYPE).reshape(-1)
    assert got.tobytes() == ref.tobytes()


def test_emission_capacity_overflow_is_esize(sx):
    from paper_2510_07868_b200 import _capi
    npx = 1000
    verts = orc.gen_vertex_tree([npx, 1500], npx)
    gv = [None] + [{k: _cuda(a) for k, a in v.items()} for v in verts[1:]]
    out = torch.zeros((100, 80), dtype=torch.uint8, device="cuda")
    with pytest.raises(_capi.NrrsError) as ei:
        sx.emit_train(gv, torch.ones((npx, 3), device="cuda"), npx, out)
    assert ei.value.code == _capi.NRRS_ESIZE


def test_film_kat_and_parity(sx):
    from paper_2510_07868_b200.film import GpuFilm
    k = json.loads((GOLDEN / "reference_kats.json").read_text())["film"]
    f = GpuFilm(k["width"], k["height"], sx)
    f.add_frame(torch.tensor(k["frame1"], dtype=torch.float64, device="cuda"))
    assert f.samples.cpu().tolist() == k["samples_after1"]
    assert f.mean_image()[0].cpu().tolist() == k["mean0_after1"]
    assert f.i_cur[1].cpu().tolist() == k["i_cur1_after1"]
    f.roll_acc()
    assert f.i_acc[0].cpu().tolist() == k["i_acc0_after_roll1"]
    f.roll_acc()
    assert f.i_acc[0].cpu().tolist() == k["i_acc0_after_roll2"]
    f.add_frame(torch.tensor(k["frame2"], dtype=torch.float64, device="cuda"))
    assert int(f.samples[0]) == k["samples0_after2"]
    assert f.mean_image()[0].cpu().tolist() == k["mean0_after2"]
    f.reset_accumulation()
    assert int(f.samples[0]) == k["samples0_after_reset"]
    assert f.i_acc[0].cpu().tolist() == k["i_acc0_after_reset"]
    # random frames: bit-exact against the oracle
    g = np.random.default_rng(2)
    npx = 1920 * 1080
    big = GpuFilm(1920, 1080, sx)
    s = np.zeros((npx, 3)); smp = np.zeros(npx, np.uint32)
    ic = np.zeros((npx, 3), np.float32); ia = np.zeros((npx, 3), np.float32)
    for _ in range(3):
        fr = g.standard_normal((npx, 3)) * 10
        big.add_frame(_cuda(fr))
        big.roll_acc()
        orc.film_add_frame(s, smp, ic, fr)
        orc.film_roll_acc(ia, ic)
    np.testing.assert_array_equal(big.sum.cpu().numpy(), s)
    np.testing.assert_array_equal(big.i_acc.cpu().numpy(), ia)
    np.testing.assert_array_equal(big.samples.cpu().numpy().view(np.uint32), smp)

"""GPU: one StatNet training step against the oracle: loss and
gradients (Mlp/HashGrid backward, FD-pinned on the oracle side), Adam + EMA bit for bit
on equal gradients, a short training sequence, and the loss-scale skip on non-finite
batches (networks.cpp:349-391, :462-552; optimizer.hpp)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as orc
from helpers import mirror_nets

pytestmark = pytest.mark.gpu


def _batch(n, seed=11):
    b = orc.gen_train_batch(n, seed)
    return b, torch.from_numpy(b.view(np.uint8).reshape(n, 80).copy()).cuda()


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


@pytest.fixture(scope="module")
def onets():
    return orc.OracleNets(orc.VARIANT_NRRS, seed=3, randomize=True)


def test_stat_loss_and_gradients_match_oracle(onets):
    from paper_2510_07868_b200.training import StatNetTrainer
    hb, db = _batch(4097)
    loss, gm, gg = orc.stat_loss(onets, hb)
    tr = StatNetTrainer(mirror_nets(onets))
    gl, fin = tr.loss_and_grad(db)
    assert fin and abs(gl - loss) <= 1e-6 * abs(loss)
    assert _rel(tr.g_mlp.cpu().numpy(), gm) < 1e-4
    assert _rel(tr.g_grid.cpu().numpy(), gg) < 1e-4
    tr.close()


def test_adam_ema_bitexact_on_equal_gradients(onets):
    from paper_2510_07868_b200.training import StatNetTrainer
    hb, _ = _batch(512)
    _, gm, gg = orc.stat_loss(onets, hb)
    tr = StatNetTrainer(mirror_nets(onets))
    theta, m, v, sh = onets.stat_mlp.copy(), np.zeros_like(gm), np.zeros_like(gm), onets.stat_mlp.copy()
    for t in (1, 2, 3):
        tr.g_mlp.copy_(torch.from_numpy(gm))
        tr._adam(tr.adam_mlp, tr.mlp, tr.g_mlp, tr.shadow_mlp, 1.0)
        orc.adam_step(theta, gm, m, v, t, 0.005)
        orc.ema_update(sh, theta, 0.99)
    np.testing.assert_array_equal(tr.mlp.cpu().numpy(), theta)
    np.testing.assert_array_equal(tr.adam_mlp.m.cpu().numpy(), m)
    np.testing.assert_array_equal(tr.adam_mlp.v.cpu().numpy(), v)
    np.testing.assert_array_equal(tr.shadow_mlp.cpu().numpy(), sh)
    tr.close()


def test_training_sequence_tracks_oracle_and_lowers_loss(onets):
    from paper_2510_07868_b200.training import StatNetTrainer
    nets = orc.OracleNets(orc.VARIANT_NRRS, seed=3, randomize=True)
    tr = StatNetTrainer(mirror_nets(nets))
    st = {k: (np.zeros_like(getattr(nets, k)), np.zeros_like(getattr(nets, k))) for k in ("stat_mlp", "stat_grid")}
    losses = []
    for step in range(1, 6):
        hb, db = _batch(8192, seed=100 + step)
        gl, applied = tr.step(db)
        loss, gm, gg = orc.stat_loss(nets, hb)
        assert applied and abs(gl - loss) <= 1e-4 * abs(loss), (step, gl, loss)
        for k, g in (("stat_mlp", gm), ("stat_grid", gg)):
            orc.adam_step(getattr(nets, k), g, st[k][0], st[k][1], step, 0.005)
        losses.append(loss)
    assert _rel(tr.mlp.cpu().numpy(), nets.stat_mlp) < 1e-3
    assert _rel(tr.grid.cpu().numpy(), nets.stat_grid) < 1e-3
    hb, db = _batch(8192, seed=100)
    assert tr.loss_and_grad(db)[0] < orc.stat_loss(orc.OracleNets(orc.VARIANT_NRRS, seed=3, randomize=True), hb,
                                                   grads=False)[0]
    tr.close()


def test_non_finite_batch_is_skipped_and_halves_the_loss_scale(onets):
    from paper_2510_07868_b200.training import StatNetTrainer
    hb, _ = _batch(300)
    hb["lo_sample"][17, 1] = np.inf
    db = torch.from_numpy(hb.view(np.uint8).reshape(300, 80).copy()).cuda()
    tr = StatNetTrainer(mirror_nets(onets))
    before = tr.mlp.clone()
    loss, applied = tr.step(db)
    assert not applied and tr.scale == 0.5 and tr.skipped_steps == 1
    assert torch.equal(tr.mlp, before)
    tr.close()


def _rrs_batch(n, seed=31, n_pixels=2048):
    b = orc.gen_train_batch(n, seed)
    g = np.random.default_rng(seed)
    b["q_real"] = (g.random(n, dtype=np.float32) * np.float32(3.0)).astype(np.float32)
    b["q_real"][::11] = 0.0
    b["q_norm"] = b["q_real"] * np.float32(0.9)
    b["k_i"] = (1 + g.integers(0, 4, n)).astype(np.float32)
    b["pixel"] = g.integers(0, n_pixels + 64, n).astype(np.uint32)  # some pixels without an error record
    b["i_pixel"] = np.float32(0.3) + g.random((n, 3), dtype=np.float32)
    return b, torch.from_numpy(b.view(np.uint8).reshape(n, 80).copy()).cuda()


@pytest.mark.parametrize("variant", [orc.VARIANT_NRRS, orc.VARIANT_AID], ids=["nrrs", "aid"])
@pytest.mark.parametrize("phase", [0, 1], ids=["warmup", "full"])
def test_rrs_loss_and_gradients_match_oracle(variant, phase):
    from paper_2510_07868_b200.training import RrsNetTrainer
    nets = orc.OracleNets(variant, seed=5, randomize=True)
    hb, db = _rrs_batch(3001)
    errors = orc.gen_pixel_errors(2048)
    parts, gm, gg = orc.rrs_loss(nets, nets.stat_grid, nets.stat_mlp, hb, errors, 0.4, phase, d_scale=0.5)
    tr = RrsNetTrainer(mirror_nets(nets))
    snap_g = torch.from_numpy(nets.stat_grid).cuda()
    snap_m = torch.from_numpy(nets.stat_mlp).cuda()
    de = torch.from_numpy(errors.view(np.float32).copy()).cuda()
    gp, sk, fin = tr.loss_and_grad(db, snap_g, snap_m, de, 0.4, phase, d_scale=0.5)
    assert fin and sk == parts.skipped
    for k in ("min", "avg", "rrs", "total"):
        ref = getattr(parts, k)
        assert abs(gp[k] - ref) <= 1e-5 * max(abs(ref), 1e-12), (k, gp[k], ref)
    assert _rel(tr.g_mlp.cpu().numpy(), gm) < 2e-4
    if variant == orc.VARIANT_AID:
        assert _rel(tr.g_grid.cpu().numpy(), gg) < 2e-4
    tr.close()


def test_grid_gradient_last_entry_with_skipped_samples():
    """The grid-gradient fold at the edges of its sorted segments: each level's LAST table entry is
    the last run of the level's segment (next to the following level's first run; keys are
    level-local, and the 0xFFFFFFFF sentinel of a slot that contributed nothing sorts after it).
    65,536 samples, so every hashed level's last entry is hit ~16 times, half of them without a
    pixel error (their pixel-error terms are skipped, hashgrid.cpp:84-103 still scatters their
    other terms): the AID grid gradient matches the oracle on those entries and overall."""
    from paper_2510_07868_b200.training import RrsNetTrainer
    nets = orc.OracleNets(orc.VARIANT_AID, seed=5, randomize=True)
    n = 1 << 16
    hb, _ = _rrs_batch(n, seed=41)
    hb["pixel"][1::2] = 4096  # no error record: skipped
    db = torch.from_numpy(hb.view(np.uint8).reshape(n, 80).copy()).cuda()
    errors = orc.gen_pixel_errors(2048)
    parts, gm, gg = orc.rrs_loss(nets, nets.stat_grid, nets.stat_mlp, hb, errors, 0.4, 1, d_scale=0.5)
    tr = RrsNetTrainer(mirror_nets(nets))
    de = torch.from_numpy(errors.view(np.float32).copy()).cuda()
    gp, sk, fin = tr.loss_and_grad(db, torch.from_numpy(nets.stat_grid).cuda(), torch.from_numpy(nets.stat_mlp).cuda(),
                                   de, 0.4, 1, d_scale=0.5)
    assert fin and sk == parts.skipped >= n // 2
    g = tr.g_grid.cpu().numpy()
    T = 1 << nets.spec.log2_table_size
    last = np.array([(lv * T + T - 1) * 2 + f for lv in range(nets.spec.levels) for f in range(2)])
    assert np.count_nonzero(gg[last]) > 0
    np.testing.assert_allclose(g[last], gg[last], rtol=1e-3, atol=1e-5 * np.abs(gg[last]).max())
    assert _rel(g, gg) < 2e-4
    tr.close()


def test_train_frame_warmup_drives_q_to_one_and_publishes():
    """NeuralRrs::train_frame in the warmup phase (q regressed to 1) + publish: the RRSNet loss
    falls and the published snapshot loads into the inference stage."""
    from paper_2510_07868_b200 import NeuralRrs, NeuralRrsConfig, RrsStage, RrsVariant, Strategy, StrategyKind
    from paper_2510_07868_b200.training import WARMUP, NeuralRrsTrainer
    nets = NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Aid, seed=1)).randomize_for_benchmark()
    tr = NeuralRrsTrainer(nets, batch=8192)
    _, db = _rrs_batch(16384, seed=9)
    first = tr.train_frame(db, None, 0.0, WARMUP)
    for _ in range(20):
        last = tr.train_frame(db, None, 0.0, WARMUP)
    assert last["loss_rrs"] < first["loss_rrs"] and last["loss_stat"] < first["loss_stat"]
    assert tr.stat.steps == 42 and tr.rrs.steps == 42
    published = tr.publish()
    st = RrsStage(4096, published)
    v = orc.gen_vertices(4096)
    out, res = st.run({k: torch.from_numpy(np.ascontiguousarray(a.view(np.int64) if a.dtype == np.uint64 else a)).cuda()
                       for k, a in v.items() if k != "pixel"}, 2, Strategy(StrategyKind.AidNrrs))
    assert np.isfinite(res.f_norm) and res.total > 0
    tr.close()


@pytest.mark.parametrize("variant", [orc.VARIANT_NRRS, orc.VARIANT_AID], ids=["nrrs", "aid"])
def test_trained_weights_stage_parity(variant):
    """Parity on TRAINED weights (every other parity test uses the x1e4-scaled
    random grids): train_frame (warmup, then the full variance-transfer phase) on the GPU, publish
    (networks.cpp:199-204), then the inference stage against the oracle holding the same snapshot:
    q_orig within the north-star 1e-3 relative, RrsRound uniforms exact, and the decisions on the
    GPU's own factors bit-exact through the oracle's decide chain."""
    from helpers import oracle_decide, rel_err
    from paper_2510_07868_b200 import NeuralRrs, NeuralRrsConfig, RateControl, RrsStage, RrsVariant, Strategy, \
        StrategyKind
    from paper_2510_07868_b200.training import FULL, WARMUP, NeuralRrsTrainer
    rv = RrsVariant.Aid if variant == orc.VARIANT_AID else RrsVariant.Nrrs
    nets = NeuralRrs(NeuralRrsConfig(variant=rv, seed=1)).randomize_for_benchmark()
    tr = NeuralRrsTrainer(nets, batch=8192)
    b, db = _rrs_batch(16384, seed=9)
    for _ in range(6):
        tr.train_frame(db, None, 0.0, WARMUP)
    errors = torch.from_numpy(orc.gen_pixel_errors(2048).view(np.float32).copy()).cuda()
    for _ in range(6):
        tr.train_frame(db, errors, 0.5, FULL)
    pub = tr.publish()
    tr.close()
    on = orc.OracleNets(variant, arrays=(pub.stat_grid, pub.stat_mlp, pub.rrs_grid, pub.rrs_mlp))
    n = 65_536
    v = orc.gen_vertices(n)
    kind = orc.AID_NRRS if variant == orc.VARIANT_AID else orc.NRRS
    from helpers import to_dev
    from paper_2510_07868_b200 import queue_capacity_for
    cap = queue_capacity_for(n)
    ref = orc.rrs_stage(v, 2, n, cap, kind, on, gain=0.85, seed=0, threads=orc.threads_available())
    st = RrsStage(n, pub)
    out, res = st.run(to_dev(v), 2, Strategy(StrategyKind(kind)), rc=RateControl(), full=True)
    torch.cuda.synchronize()
    q = out.q_orig.cpu().numpy()
    assert np.all(np.isfinite(q))
    err = rel_err(q, ref["q_orig"], 1e-6)
    assert err.max() <= 1e-3, f"trained-weight q_orig max rel err {err.max():.3e}"
    np.testing.assert_array_equal(out.u.cpu().numpy(), ref["u"])
    dec = oracle_decide(q, out.u.cpu().numpy(), n, cap, 0.85)
    np.testing.assert_array_equal(out.k.cpu().numpy(), dec["k"])
    np.testing.assert_array_equal(out.slots.cpu().numpy()[:res.spawned].view(np.uint32), dec["slots"])
    st.close()


@pytest.mark.parametrize("variant", [orc.VARIANT_NRRS, orc.VARIANT_AID], ids=["nrrs", "aid"])
def test_training_is_bitwise_deterministic(variant):
    """Two identical train_frame sequences (warmup then full phase) from the same nets give
    bitwise-identical live weights, EMA snapshots and losses (the reference's neural runs are
    bit-identical across runs, test_harness.cpp:370-403): the hash-grid gradient scatter is a
    stable sort by entry + in-order run sums, not float atomics."""
    from paper_2510_07868_b200 import NeuralRrs, NeuralRrsConfig, RrsVariant
    from paper_2510_07868_b200.training import FULL, WARMUP, NeuralRrsTrainer
    rv = RrsVariant.Aid if variant == orc.VARIANT_AID else RrsVariant.Nrrs
    _, db = _rrs_batch(20000, seed=4)
    errors = torch.from_numpy(orc.gen_pixel_errors(2048).view(np.float32).copy()).cuda()
    runs = []
    for _ in range(2):
        nets = NeuralRrs(NeuralRrsConfig(variant=rv, seed=1)).randomize_for_benchmark()
        tr = NeuralRrsTrainer(nets, batch=8192)
        losses = [tr.train_frame(db, None, 0.0, WARMUP) for _ in range(3)]
        losses += [tr.train_frame(db, errors, 0.5, FULL) for _ in range(3)]
        pub = tr.publish()
        runs.append(([np.asarray(x).copy() for x in (pub.stat_grid, pub.stat_mlp, pub.rrs_grid, pub.rrs_mlp)],
                     losses))
        tr.close()
    (wa, la), (wb, lb) = runs
    for x, y in zip(wa, wb):
        assert x.tobytes() == y.tobytes()
    assert la == lb


@pytest.mark.parametrize("variant", [orc.VARIANT_NRRS, orc.VARIANT_AID], ids=["nrrs", "aid"])
def test_non_default_grid_runs_the_generic_training_kernels(variant):
    """3 levels, base 4, 2^10 entries: StatNet input 22, so the steps take the generic (runtime-width)
    kernels and the scatter sorts 11-bit entry segments; gradients still match the oracle."""
    from paper_2510_07868_b200.training import RrsNetTrainer, StatNetTrainer
    nets = orc.OracleNets(variant, levels=3, base=4, log2t=10, seed=9, randomize=True)
    hb, db = _batch(2049, seed=4)
    loss, gm, gg = orc.stat_loss(nets, hb)
    tr = StatNetTrainer(mirror_nets(nets))
    gl, fin = tr.loss_and_grad(db)
    assert fin and abs(gl - loss) <= 1e-6 * abs(loss)
    assert _rel(tr.g_mlp.cpu().numpy(), gm) < 1e-4
    assert _rel(tr.g_grid.cpu().numpy(), gg) < 1e-4
    tr.close()
    hb2, db2 = _rrs_batch(2049)
    errors = orc.gen_pixel_errors(2048)
    parts, gm2, gg2 = orc.rrs_loss(nets, nets.stat_grid, nets.stat_mlp, hb2, errors, 0.4, 1, d_scale=0.5)
    rt = RrsNetTrainer(mirror_nets(nets))
    gp, sk, fin = rt.loss_and_grad(db2, torch.from_numpy(nets.stat_grid).cuda(),
                                   torch.from_numpy(nets.stat_mlp).cuda(),
                                   torch.from_numpy(errors.view(np.float32).copy()).cuda(), 0.4, 1, d_scale=0.5)
    assert fin and sk == parts.skipped
    assert abs(gp["total"] - parts.total) <= 1e-5 * max(abs(parts.total), 1e-12)
    assert _rel(rt.g_mlp.cpu().numpy(), gm2) < 2e-4
    if variant == orc.VARIANT_AID:
        assert _rel(rt.g_grid.cpu().numpy(), gg2) < 2e-4
    rt.close()

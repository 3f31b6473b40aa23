"""CPU: the host mirror of the reference interface (rrs.hpp, networks.hpp) and the
C ABI library's load / export contract.  No device calls."""
from __future__ import annotations

import ctypes as C
import os
import pathlib
import re
import subprocess

import numpy as np
import pytest

import oracle as orc
from paper_2510_07868_b200 import (HashGridSpec, NeuralRrs, NeuralRrsConfig, RrsVariant, Strategy, StrategyKind,
                                   assignment_name, parse_assignment, parse_strategy, strategy_name, synthetic)
from paper_2510_07868_b200 import _capi
from paper_2510_07868_b200.sharded import f_norm_from_sums, global_clip

ROOT = pathlib.Path(__file__).resolve().parents[1]


# ---------------------------------------------------------------- ABI -------
def header_functions():
    text = (ROOT / "include" / "nrrs_gpu.h").read_text()
    return re.findall(r"NRRS_API\s+[\w\s\*]+?\b(nrrs_\w+)\s*\(", text)


def test_library_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 20
    lib = _capi.lib()
    for n in names:
        assert hasattr(lib, n), n
    bound = {s[0] for s in _capi.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound
    out = subprocess.run(["nm", "-D", "--defined-only", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (nrrs_\w+)", out))
    assert set(names) <= exported


def test_library_is_sm100a_tcgen05_code():
    sass = subprocess.run(["cuobjdump", "-sass", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "LDTM" in sass and "STTM" in sass  # tcgen05.ld / tcgen05.st
    elf = subprocess.run(["cuobjdump", "-lelf", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in elf


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    h = C.c_void_p()
    assert _capi.lib().nrrs_gpu_create(0, C.byref(h)) == _capi.NRRS_ECUDA
    from paper_2510_07868_b200 import RrsStage
    with pytest.raises(RuntimeError):
        RrsStage(16)


def test_product_never_imports_the_oracle():
    pkg = ROOT / "paper_2510_07868_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.h")) + list(pkg.rglob("*.cuh")):
        text = f.read_text()
        assert "import oracle" not in text and "liborc" not in text and "nrrs_oracle" not in text, f


def test_abi_version_and_host_helpers():
    lib = _capi.lib()
    assert lib.nrrs_gpu_abi_version() == 1
    assert lib.nrrs_queue_capacity_for(14400) == 16200
    assert lib.nrrs_root_path_key(0, 0) == 0xE220A8397B1DCDAF


# ------------------------------------------------------------ rrs.hpp -------
def test_strategy_parsing_round_trip():
    """test_rrs.cpp:135-154."""
    assert parse_strategy("fixed:0.5").fixed_value == pytest.approx(0.5)
    assert parse_strategy("fixed").fixed_value == 1.0
    assert parse_strategy("pt").kind == StrategyKind.Fixed
    for name, kind in (("throughput", StrategyKind.Throughput), ("adrrs-tree", StrategyKind.AdrrsTree),
                       ("adrrs-nn", StrategyKind.AdrrsNn), ("nrrs", StrategyKind.Nrrs),
                       ("aid-nrrs", StrategyKind.AidNrrs)):
        assert parse_strategy(name).kind == kind
        assert strategy_name(parse_strategy(name)) == name
    with pytest.raises(RuntimeError):
        parse_strategy("bogus")
    with pytest.raises(RuntimeError):
        parse_strategy("fixed:-1")
    a = parse_assignment("nrrs,adrrs-nn,fixed:1", 3)
    assert [s.kind for s in a] == [StrategyKind.Nrrs, StrategyKind.AdrrsNn, StrategyKind.Fixed]
    with pytest.raises(RuntimeError):
        parse_assignment("nrrs,nrrs", 3)
    u = parse_assignment("throughput", 4)
    assert assignment_name(u) == "throughput,throughput,throughput,throughput"
    assert strategy_name(Strategy(StrategyKind.Fixed, 2.5)) == "fixed:2.5"
    assert Strategy(StrategyKind.Nrrs).neural() and not Strategy(StrategyKind.Fixed).adaptive()


# -------------------------------------------------------- networks.hpp ------
@pytest.mark.parametrize("variant", [RrsVariant.Nrrs, RrsVariant.Aid])
@pytest.mark.parametrize("grid", [(8, 2, 16, 15), (3, 2, 4, 10)])
def test_neural_rrs_init_matches_reference_constructor(variant, grid):
    """NeuralRrs() reproduces networks.cpp:159-197 bit for bit (oracle restatement)."""
    cfg = NeuralRrsConfig(variant=variant, grid=HashGridSpec(*grid), seed=77)
    host = NeuralRrs(cfg)
    ref = orc.OracleNets(int(variant), *grid, seed=77, randomize=False)
    np.testing.assert_array_equal(host.stat_grid, ref.stat_grid)
    np.testing.assert_array_equal(host.stat_mlp, ref.stat_mlp)
    np.testing.assert_array_equal(host.rrs_grid, ref.rrs_grid)
    np.testing.assert_array_equal(host.rrs_mlp, ref.rrs_mlp)
    host.randomize_for_benchmark()
    ref = orc.OracleNets(int(variant), *grid, seed=77, randomize=True)
    for a, b in ((host.stat_grid, ref.stat_grid), (host.stat_mlp, ref.stat_mlp), (host.rrs_grid, ref.rrs_grid),
                 (host.rrs_mlp, ref.rrs_mlp)):
        np.testing.assert_array_equal(a, b)


def test_param_counts_match_reference():
    assert NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Nrrs)).stat_mlp.size == 3366
    assert NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Nrrs)).rrs_mlp.size == 2529
    assert NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Aid)).rrs_mlp.size == 3201
    assert NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Nrrs)).rrs_grid.size == 0


def test_checkpoint_round_trip_and_mismatch(tmp_path):
    """NRRSCK01 (networks.cpp:610-705); test_networks.cpp:936-986 behaviour."""
    cfg = NeuralRrsConfig(variant=RrsVariant.Aid, grid=HashGridSpec(3, 2, 4, 10), seed=65)
    a = NeuralRrs(cfg).randomize_for_benchmark()
    path = str(tmp_path / "ck.bin")
    a.save_checkpoint(path)
    b = NeuralRrs(cfg)
    b.load_checkpoint(path)
    for x, y in ((a.stat_grid, b.stat_grid), (a.stat_mlp, b.stat_mlp), (a.rrs_grid, b.rrs_grid),
                 (a.rrs_mlp, b.rrs_mlp)):
        np.testing.assert_array_equal(x, y)
    # a reference-layout file: magic, version, variant, spec, dims, 12 blocks, adam, scalars
    data = pathlib.Path(path).read_bytes()
    assert data[:8] == b"NRRSCK01"
    other = NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Nrrs, grid=HashGridSpec(3, 2, 4, 10), seed=65))
    with pytest.raises(RuntimeError):
        other.load_checkpoint(path)
    pathlib.Path(path).write_bytes(data[:100])
    with pytest.raises(RuntimeError):
        b.load_checkpoint(path)


def test_synthetic_generator_matches_oracle():
    a = orc.gen_vertices(3000, 1000, 5)
    b = synthetic.gen_vertices(3000, n_pixels=1000, frame=5)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])
    np.testing.assert_array_equal(orc.split_bound_factors(777), synthetic.split_bound_factors(777))
    # bands for the tile-sharded layout concatenate to the global batch
    full = synthetic.gen_vertices(2000, n_pixels=2000)
    band = synthetic.gen_vertices(1000, n_pixels=2000, first=1000)
    for k in full:
        np.testing.assert_array_equal(full[k][1000:], band[k])


# ------------------------------------------------------------ sharding ------
def test_global_clip_arithmetic():
    # no overflow
    assert global_clip([3, 4, 5], 1, 100) == (3, 4, 12, 0)
    # overflow lands in the middle rank: ranks after it keep nothing
    tot = [60, 50, 30]
    got = [global_clip(tot, r, 100) for r in range(3)]
    assert [g[1] for g in got] == [60, 40, 0]
    assert all(g[2] == 100 and g[3] == 40 for g in got)
    # same as plan_spawns on the concatenated queue
    counts = np.concatenate([np.full(t, 1, np.int32) for t in tot])
    off, sp, dr = orc.plan_spawns(counts, 100)
    assert (sp, dr) == (100, 40)
    assert f_norm_from_sums([1.0, 2.0, 1.0], 2) == pytest.approx(0.5)
    assert f_norm_from_sums([0.0, 0.0], 7) == 1.0

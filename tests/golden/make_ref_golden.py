"""Regenerate ref_nets_golden.npz from the REFERENCE's own networks.cpp / mlp.cpp / hashgrid.cpp.

oracle/_ref/libref_nets.so is compiled by oracle/Makefile (target `ref`) from the reference sources
unmodified, against the Eigen subset shim in oracle/eigen_shim.  The nets are the benchmark's
random-init snapshots (OracleNets(variant, seed=1, randomize=True)), handed to the
reference through a NRRSCK01 checkpoint written by this repo's NeuralRrs.save_checkpoint and read
by the reference's NeuralRrs::load_checkpoint (networks.cpp:641-705), so the fixture also pins the
checkpoint interchange.  Outputs: predict_q and predict_stats on 1,024 SURVEY.md 8d vertices per
variant.  Run from the repo root (needs /root/reference; the fixture itself travels):
    make -C oracle ref && python tests/golden/make_ref_golden.py
"""
import ctypes as C
import pathlib
import sys
import tempfile

import numpy as np

root = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(root))
sys.path.insert(0, str(root / "tests"))
import oracle as orc  # noqa: E402
from helpers import mirror_nets  # noqa: E402

N = 1024
lib = C.CDLL(str(root / "oracle/_ref/libref_nets.so"))
lib.ref_predict.restype = C.c_int
lib.ref_predict.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_size_t] + [C.c_void_p] * 7
v = orc.gen_vertices(N)
out = {"p01": v["p01"], "wo01": v["wo01"], "roughness": v["roughness"], "weight": v["weight"],
       "i_pixel": v["i_pixel"], "path_key": v["path_key"]}
for name, variant in (("nrrs", orc.VARIANT_NRRS), ("aid", orc.VARIANT_AID)):
    on = orc.OracleNets(variant, seed=1, randomize=True)
    with tempfile.TemporaryDirectory() as d:
        ck = str(pathlib.Path(d) / "nets.ck")
        mirror_nets(on).save_checkpoint(ck)
        q = np.zeros(N, np.float32)
        st = np.zeros((N, 6), np.float32)
        s = on.spec
        rc = lib.ref_predict(ck.encode(), variant, s.levels, s.features, s.base_resolution, s.log2_table_size, N,
                             v["p01"].ctypes.data, v["wo01"].ctypes.data, v["roughness"].ctypes.data,
                             v["weight"].ctypes.data, v["i_pixel"].ctypes.data, q.ctypes.data, st.ctypes.data)
        assert rc == 0, f"reference rejected the checkpoint ({name})"
    out[f"{name}_q"] = q
    out[f"{name}_stats"] = st
np.savez_compressed(root / "tests/golden/ref_nets_golden.npz", **out,
                    _source=np.array("reference networks.cpp/mlp.cpp/hashgrid.cpp compiled unmodified "
                                     "(oracle/eigen_shim), OracleNets(seed=1, randomize=True) via NRRSCK01"))
print("wrote", N, "vertices x 2 variants")

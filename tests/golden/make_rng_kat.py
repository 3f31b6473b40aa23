"""Regenerate rng_kat.json from the reference's own rng.hpp.

oracle/_ref/rng_kat is compiled by oracle/Makefile (target `ref`) from
/root/reference/proj/include/nrrs/rng.hpp verbatim plus the driver
oracle/ref_rng_kat.cpp.  Run from the repo root:
    make -C oracle ref && python tests/golden/make_rng_kat.py
"""
import json
import pathlib
import subprocess

root = pathlib.Path(__file__).resolve().parents[2]
out = subprocess.run([str(root / "oracle/_ref/rng_kat")], check=True, capture_output=True, text=True).stdout
data = json.loads(out)
data["_source"] = "reference proj/include/nrrs/rng.hpp compiled verbatim (oracle/ref_rng_kat.cpp driver)"
(root / "tests/golden/rng_kat.json").write_text(json.dumps(data, indent=1) + "\n")
print("wrote", len(data["pixels"]), "pixel KATs")

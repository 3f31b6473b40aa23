"""Driver for the configs[1] render (NRRS, builtin Cornell 512x512, B = 12): wall ms per frame, for
comparing against an ncu launch list of the same command.
usage: python tools/prof_render.py [frames]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2510_07868_b200 import (NeuralRrs, NeuralRrsConfig, RateControl, RrsStage, RrsVariant, Strategy,
                                   StrategyKind)
from paper_2510_07868_b200 import render as rnd
from paper_2510_07868_b200.film import GpuFilm, SuffixStage

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w, h, B = 512, 512, 12
nets = NeuralRrs(NeuralRrsConfig(variant=RrsVariant.Nrrs, seed=1)).randomize_for_benchmark()
st = RrsStage(w * h, nets)
sc = rnd.GpuScene(rnd.make_cornell_scene(), ctx=st.ctx)
tr = rnd.Tracer(sc, w * h, B)
film = GpuFilm(w, h, SuffixStage(ctx=st.ctx))
assign = [Strategy()] + [Strategy(StrategyKind.Nrrs)] * (B - 1)
rc = RateControl()
for f in range(2):
    tr.trace_frame(assign, rnd.TraceConfig(max_depth=B, seed=11, frame_index=f), rc, film)
    film.roll_acc()
torch.cuda.synchronize()
t0 = time.perf_counter()
for f in range(frames):
    tr.trace_frame(assign, rnd.TraceConfig(max_depth=B, seed=11, frame_index=2 + f), rc, film)
    film.roll_acc()
torch.cuda.synchronize()
print(f"configs1: {1e3 * (time.perf_counter() - t0) / frames:.3f} ms/frame over {frames} frames")

"""Precision simulation of the AID RRSNet forward (Precision): worst-case relative
error of q for the 3-term fp16 split, the two 2-term variants and plain fp16, against an fp64 forward
on SURVEY.md 8d vertices with the bench snapshot (fp16 grid tables in every variant).  CPU only.
usage: python tools/precision_sim.py [n_vertices] [hidden_weight_scale]"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)
import oracle as orc
L=orc.lib()
L.orc_build_aid_tail.argtypes=[C.c_void_p,C.c_void_p,C.c_void_p,C.c_float,C.c_void_p]
N=int(sys.argv[1]) if len(sys.argv)>1 else 100000
scale=float(sys.argv[2]) if len(sys.argv)>2 else 1.0
on=orc.OracleNets(orc.VARIANT_AID, seed=1, randomize=True)
v=orc.gen_vertices(N)
# layer-0 input: grid features (fp16 table) + tail
theta16=on.rrs_grid.astype(np.float16).astype(np.float32)
X=np.zeros((N,32),np.float32)
for i in range(N):
    L.orc_grid_encode(C.byref(on.spec), theta16.ctypes.data, v["p01"][i].ctypes.data, X[i].ctypes.data)
    L.orc_build_aid_tail(v["wo01"][i].ctypes.data, v["weight"][i].ctypes.data, v["i_pixel"][i].ctypes.data, float(v["roughness"][i]), X[i,16:].ctypes.data)
th=on.rrs_mlp.copy()
# layers
dims=[(32,32),(32,32),(32,32),(32,1)]
Ws=[];Bs=[];off=0
for li,lo in dims:
    W=th[off:off+li*lo].reshape(li,lo).T.astype(np.float64); off+=li*lo
    b=th[off:off+lo].astype(np.float64); off+=lo
    Ws.append(W*(scale if lo>1 else 1.0)); Bs.append(b)
def f16(a): return a.astype(np.float16).astype(np.float64)
def split(a): h=f16(a); return h, f16(a-h)
def fwd(mode):
    a=X.astype(np.float64)
    for l,(W,b) in enumerate(zip(Ws,Bs)):
        Wh,Wl=split(W)
        if mode=='exact': z=a@W.T
        elif mode=='s3': ah,al=split(a); z=ah@Wh.T+al@Wh.T+ah@Wl.T
        elif mode=='s2a': ah=f16(a); z=ah@Wh.T+ah@Wl.T      # A rounded, W exact
        elif mode=='s2w': ah,al=split(a); z=ah@Wh.T+al@Wh.T # A exact, W rounded
        elif mode=='p16': z=f16(a)@Wh.T
        z=(z+b).astype(np.float32).astype(np.float64)
        if l<3: a=np.maximum(z,0.01*z)
        else: y=z[:,0]
    return np.where(y<0, np.log1p(np.exp(y)), 0.5*y+np.log(2.0))
ref=fwd('exact')
for m in ['s3','s2a','s2w','p16']:
    q=fwd(m); e=np.abs(q-ref)/np.abs(ref)
    print(f"scale {scale} {m:4s} max {e.max():.2e} p99.99 {np.quantile(e,0.9999):.2e} mean {e.mean():.2e}")

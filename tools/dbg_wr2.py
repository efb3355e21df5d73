import numpy as np, sys
sys.path.insert(0,'/root/repo')
from tests.fixtures import load
from paper_2007_08576_b200 import kernels as K
kz = load("kernels")
c = 18
sl = slice(c, c+1)
base = dict(gate=8.0, cg=float(np.cos(np.deg2rad(60.0))), dv=kz["wr_valid_px"], on=kz["wr_obs_normals"])
def run(**kw):
    a = {**base, **kw}
    got = K.warp_and_rasterize(kz["wr_points"][sl], kz["normals"][sl], kz["bind_idx"][sl], kz["alpha"][sl], kz["warps"], kz["wr_depth"], a["dv"], a["on"], 120.0, 120.0, 23.5, 23.5, a["gate"], a["cg"], 8)
    return got[2][0], got[5][0]
print("base", run())
print("dvalid all", run(dv=np.ones((48,48), bool)))
print("gate big", run(gate=1e9))
print("cos -1", run(cg=-1.0))
print("all relaxed", run(dv=np.ones((48,48), bool), gate=1e9, cg=-1.0))
print("dvalid at", kz["wr_valid_px"][30,19], kz["wr_depth"][30,19], kz["wr_obs_normals"][30,19])

import numpy as np, sys
sys.path.insert(0,'/root/repo')
from tests.fixtures import load
from paper_2007_08576_b200 import kernels as K
kz = load("kernels")
got = K.warp_and_rasterize(kz["wr_points"], kz["normals"], kz["bind_idx"], kz["alpha"], kz["warps"], kz["wr_depth"], kz["wr_valid_px"], kz["wr_obs_normals"], 120.0, 120.0, 23.5, 23.5, 8.0, float(np.cos(np.deg2rad(60.0))), 8)
names = ("p","n","valid","obs_p","obs_n","pixels")
for g, nm in zip(got, names):
    ref = kz["wr_"+nm]
    bad = np.flatnonzero((g != ref).reshape(len(g), -1).any(axis=1))
    print(nm, "mismatch rows", bad[:10], np.abs(g.astype(float)-ref.astype(float)).max())
c = 18
print("gpu p", got[0][c], "ref", kz["wr_p"][c]); print("gpu n", got[1][c], "ref", kz["wr_n"][c]); print("pix", got[5][c], kz["wr_pixels"][c])

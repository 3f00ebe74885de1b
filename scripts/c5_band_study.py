"""Host sweep over a plan's tiles and interior views: staged quad bytes per voxel-view update of the
window kernel's full-column boxes vs per-slice row bands (union of a tile's open slices per view,
3 quad rows each). Usage: python scripts/c5_band_study.py C5"""
import numpy as np, sys
import os; sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
from synth import configs
import paper_2201_02309_b200 as k
name = sys.argv[1] if len(sys.argv)>1 else 'C5'
cfg = configs.get(name)
plan = k.Plan(cfg, device=-1); plan.precompute()
T = plan.export_tables()
pf, pl = T['pi_first'], T['pi_last']
nz, ny, nx = pf.shape
R, D, dw, da, nr, nc = cfg['R'], cfg['D'], cfg['d_w'], cfg['d_alpha'], cfg['n_rows'], cfg['n_cols']
dlam = 2*np.pi/cfg['views_per_turn']; h = cfg['P']/(2*np.pi); dz = cfg['P']/nz
dx = cfg['dx']; aoff = cfg['alpha_offset']
TX=TY=16
row_c15 = 0.5*(nr-1)+1.5
nbmax=0; hist={}; spanh={}; upd=0; bytes3=0; bytescur=0; cnt=0
for ty in range(ny//TY):
  for tx in range(nx//TX):
    xa=(tx*TX-0.5*nx)*dx; xb=xa+(TX-1)*dx; ya=(ty*TY-0.5*ny)*dx; yb=ya+(TY-1)*dx
    a = pf[:, ty*TY:(ty+1)*TY, tx*TX:(tx+1)*TX]+1; b = pl[:, ty*TY:(ty+1)*TY, tx*TX:(tx+1)*TX]-1
    ok = a<=b
    if not ok.any(): continue
    Kf = np.where(ok, a, 1<<30).reshape(nz,-1).min(1); Kl = np.where(ok, b, -(1<<30)).reshape(nz,-1).max(1)
    k0 = Kf.min(); k1 = Kl.max()
    cx=np.array([xa,xb,xa,xb]); cy=np.array([ya,ya,yb,yb])
    for kk in range(k0,k1+1):
        lam = kk*dlam + cfg['lambda0']; c,s=np.cos(lam),np.sin(lam)
        vs = R - cx*c - cy*s; us = -cx*s + cy*c
        col = np.arctan2(us,vs)/da + 0.5*(nc-1) - aoff
        bw = int(np.floor(col.max())-np.floor(col.min()))+3
        sc = D/np.hypot(us,vs)/dw
        js = np.nonzero((Kf<=kk)&(kk<=Kl))[0]
        nb = len(js); nbmax=max(nbmax,nb); hist[nb]=hist.get(nb,0)+1
        zs = cfg['z0']+h*kk*dlam
        for j in js:
            p = sc*(j*dz - zs) + row_c15
            r0 = np.floor(p.min()-0.02+0.5); r1 = np.floor(p.max()+0.02+0.5)
            sp = int(r1-r0+1); spanh[sp]=spanh.get(sp,0)+1
        upd += (ok & (a<=kk) & (kk<=b)).sum()
        bytes3 += nb*bw*3*16; bytescur += bw*19*16
print(name, "nbmax", nbmax, "hist", sorted(hist.items()), "span", sorted(spanh.items()))
print("B/upd cur", bytescur/upd, "band3", bytes3/upd)

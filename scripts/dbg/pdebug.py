import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))

import numpy as np, torch
from test_gpu_pencil_virtual import _case, M
from paper_1309_2451_b200 import _lib, qgrid
from paper_1309_2451_b200.pencil import PencilLayout
from paper_1309_2451_b200.propagator import NativePlan
from oracle import split_step as orc
n=(32,16,32); Pr=Pc=2; P=4
grid, v, a0 = _case(n)
f = orc.make_factors(orc.as_grid(grid), v, M, 1e-6)
lays=[PencilLayout(grid.n,Pr,Pc,r) for r in range(P)]
plans=[]; bufs=[]
for lay in lays:
    vb=torch.from_numpy(np.ascontiguousarray(v[lay.x_slice, lay.y_slice])).cuda()
    plans.append(NativePlan(grid, vb, M, 1e-6, slab_p=P, slab_r=lay.rank, pencil_c=Pc))
    b={k: torch.empty(lay.points, dtype=torch.complex128, device='cuda') for k in ('zc','yb','xp','xr')}
    b['psi']=torch.from_numpy(np.ascontiguousarray(a0[lay.x_slice, lay.y_slice])).cuda().reshape(-1)
    bufs.append(b)
def a2a(which, src, dst):
    groups=[lays[a*Pc].row_ranks() for a in range(Pr)] if which=='row' else [lays[b].col_ranks() for b in range(Pc)]
    for members in groups:
        G=len(members); chunk=lays[0].points//G
        for qi,q in enumerate(members):
            for pi,p in enumerate(members):
                bufs[q][dst][pi*chunk:(pi+1)*chunk].copy_(bufs[p][src][qi*chunk:(qi+1)*chunk])
nx,ny,nz=n
# global reference stages
g0 = np.fft.fft(a0*f.exp_v_half, axis=2)
g1 = np.fft.fft(g0, axis=1)
g2 = np.fft.ifft(np.fft.fft(g1, axis=0)*f.exp_k, axis=0)
def chk(name, got, ref):
    print(name, float(np.abs(got-ref).max()/np.abs(ref).max()))
for r in range(P): plans[r].run_pass(_lib.PASS_PZ_FIRST, bufs[r]['psi'], bufs[r]['zc'])
for r,lay in enumerate(lays):
    blk=g0[lay.x_slice, lay.y_slice]  # (xa,yb,nz)
    zc=blk.reshape(lay.xa,lay.yb,Pc,lay.zc).transpose(2,0,1,3).reshape(-1)
    chk(f'zc r{r}', bufs[r]['zc'].cpu().numpy(), zc)
a2a('row','zc','yb')
for r,lay in enumerate(lays):
    zsl=slice(lay.b*lay.zc,(lay.b+1)*lay.zc)
    blk=g0[lay.x_slice, :, zsl]  # (xa, ny, zc)
    yb=blk.reshape(lay.xa,Pc,lay.yb,lay.zc).transpose(1,0,2,3).reshape(-1)
    chk(f'yb r{r}', bufs[r]['yb'].cpu().numpy(), yb)
for r in range(P): plans[r].run_pass(_lib.PASS_PY_FWD, bufs[r]['yb'], bufs[r]['xp'])
for r,lay in enumerate(lays):
    zsl=slice(lay.b*lay.zc,(lay.b+1)*lay.zc)
    blk=g1[lay.x_slice, :, zsl]
    xp=blk.reshape(lay.xa,Pr,lay.yd,lay.zc).transpose(1,0,2,3).reshape(-1)
    chk(f'xp r{r}', bufs[r]['xp'].cpu().numpy(), xp)
a2a('col','xp','xr')
for r,lay in enumerate(lays):
    zsl=slice(lay.b*lay.zc,(lay.b+1)*lay.zc); ysl=slice(lay.a*lay.yd,(lay.a+1)*lay.yd)
    chk(f'xr r{r}', bufs[r]['xr'].cpu().numpy(), g1[:, ysl, zsl].reshape(-1))
for r in range(P): plans[r].run_pass(_lib.PASS_PX_KIN, bufs[r]['xr'], bufs[r]['xr'])
for r,lay in enumerate(lays):
    zsl=slice(lay.b*lay.zc,(lay.b+1)*lay.zc); ysl=slice(lay.a*lay.yd,(lay.a+1)*lay.yd)
    chk(f'xk r{r}', bufs[r]['xr'].cpu().numpy(), g2[:, ysl, zsl].reshape(-1)/ (nx*ny*nz) * 1.0)
g2 = g2 * nx / (nx*ny*nz)
a2a('col','xr','xp')
for r,lay in enumerate(lays):
    zsl=slice(lay.b*lay.zc,(lay.b+1)*lay.zc)
    blk=g2[lay.x_slice, :, zsl]
    xp=blk.reshape(lay.xa,Pr,lay.yd,lay.zc).transpose(1,0,2,3).reshape(-1)
    chk(f'xp2 r{r}', bufs[r]['xp'].cpu().numpy(), xp)
for r in range(P): plans[r].run_pass(_lib.PASS_PY_INV, bufs[r]['xp'], bufs[r]['yb'])
g3 = np.fft.ifft(g2, axis=1)*ny
for r,lay in enumerate(lays):
    zsl=slice(lay.b*lay.zc,(lay.b+1)*lay.zc)
    blk=g3[lay.x_slice, :, zsl]
    yb=blk.reshape(lay.xa,Pc,lay.yb,lay.zc).transpose(1,0,2,3).reshape(-1)
    chk(f'yb2 r{r}', bufs[r]['yb'].cpu().numpy(), yb)
a2a('row','yb','zc')
for r,lay in enumerate(lays):
    blk=g3[lay.x_slice, lay.y_slice]
    zc=blk.reshape(lay.xa,lay.yb,Pc,lay.zc).transpose(2,0,1,3).reshape(-1)
    chk(f'zc2 r{r}', bufs[r]['zc'].cpu().numpy(), zc)
for r in range(P): plans[r].run_pass(_lib.PASS_PZ_LAST, bufs[r]['zc'], bufs[r]['psi'])
g4 = np.fft.ifft(g3, axis=2)*nz*f.exp_v_half
for r,lay in enumerate(lays):
    chk(f'psi r{r}', bufs[r]['psi'].cpu().numpy(), g4[lay.x_slice, lay.y_slice].reshape(-1))

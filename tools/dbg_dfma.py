import sys; sys.path.insert(0,'.')
import numpy as np, torch, oracle
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors, synthetic_q_np
for (n,nbw,nev,ldq) in [(97,8,9,100),(97,8,9,98),(97,8,64,98),(301,8,45,302),(97,16,9,100),(200,8,9,200)]:
    s,L=oracle.schedule(n,nbw); hv,tau=synthetic_reflectors(len(s),nbw,17+n); Q=synthetic_q_np(n,0,nev,17+n,ldq=ldq)
    want=oracle.apply(hv,tau,s,L,Q)
    for grid in (0,1):
        for kf in (2,8):
            dq=torch.from_numpy(Q.copy()).cuda()
            eb.trans_ev_tridi_to_band(n,nbw,torch.from_numpy(hv).cuda(),torch.from_numpy(tau).cuda(),dq,opts=dict(kernel=3,fused_k=kf,grid_ctas=grid))
            got=dq.cpu().numpy()
            err=np.abs(got[:,:n]-want[:,:n]).max()
            bad=np.argwhere(np.abs(got[:,:n]-want[:,:n])>1e-10)
            print(n,nbw,nev,ldq,grid,kf,err, bad[:5].tolist(), flush=True)

"""Culling simulation (numpy): (group, source) slot steps per rotation with
32-point reference groups vs half- / quarter-warp sub-groups (each warp step
waiting for its longest sub-list), on the bench pairs at random rotations.
    python tools/cull_sim.py c2|c4"""
import numpy as np, math, sys
cfg=sys.argv[1] if len(sys.argv)>1 else 'c2'
d=np.load(f'/root/repo/bench_data/benchgen_{cfg}.npz')
x=d['x0']; y=d['y0']
if cfg=='c4': bin_=0.004; k=4; amp=math.radians(5)
else: bin_=0.025; k=20; amp=math.pi/4
W=(2*k+1)*bin_
def kd(idx, pts, G):
    if len(idx)<=G: return [idx]
    sub=pts[idx]; ax=np.argmax(sub.max(0)-sub.min(0))
    o=idx[np.argsort(sub[:,ax],kind='stable')]
    nt=(len(idx)+G-1)//G; left=(nt//2)*G
    return kd(o[:left],pts,G)+kd(o[left:],pts,G)
def rot(a,b,c):
    ca,sa,cb,sb,cc,sc=math.cos(a),math.sin(a),math.cos(b),math.sin(b),math.cos(c),math.sin(c)
    Rx=np.array([[1,0,0],[0,ca,-sa],[0,sa,ca]]);Ry=np.array([[cb,0,sb],[0,1,0],[-sb,0,cb]]);Rz=np.array([[cc,-sc,0],[sc,cc,0],[0,0,1]])
    return Rz@Ry@Rx
rng=np.random.default_rng(1)
lo=-k*bin_-bin_/2
g32=kd(np.arange(len(y)),y,32)
halves=[kd(g,y,16) for g in g32]
quarters=[[q for h in kd(g,y,16) for q in kd(h,y,8)] for g in g32]
units=kd(np.arange(len(x)),x,32)
def passes(Y, p):
    blo=Y.min(0); bhi=Y.max(0)
    return np.all((bhi-p>=lo)&(blo-p<lo+W),axis=1)
nr=10; s32=s16=s8=nunits=0
for r in range(nr):
    R=rot(*rng.uniform(-amp,amp,3)); p=x@R.T
    for gi,g in enumerate(g32):
        for u in units:
            pu=p[u]
            # unit box cull
            ulo=pu.min(0); uhi=pu.max(0); Y=y[g]
            if not np.all((Y.max(0)-ulo>=lo)&(Y.min(0)-uhi<lo+W)): continue
            nunits+=1
            s32+=passes(Y,pu).sum()
            s16+=max(passes(y[h],pu).sum() for h in halves[gi])
            s8+=max(passes(y[q],pu).sum() for q in quarters[gi])
print(cfg, 'units/rot', nunits/nr, 'steps32', s32/nr, 'steps16(max)', s16/nr, 'steps8(max)', s8/nr)

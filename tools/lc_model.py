"""Developer model (CPU): candidates staged per interaction by the fused kernel's
row trimming on the real config-3 cloud, for a patch of queries grouped in
Morton order.  Prints, relative to the exact neighbourhood sizes:
  union/exact    the staged union of a group's row chords (what the kernel pays),
  perquery/exact each query's own trimmed rows (the quantisation alone),
  maxper/exact   the longest per-query list in a group,
  and the pair-union figures for 2-query sub-groups.

    python tools/lc_model.py [G]        # G queries per group (default 8)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_03365_b200 as pb
from scipy.spatial import cKDTree
P, X = pb.generate_config(3, 1.0)
P = P.astype(np.float32).astype(np.float64); X = X.astype(np.float32).astype(np.float64)
s = 0.02
# patch
c = np.array([0.3, -0.2])
def inpatch(A, r): return (np.abs(A[:,0]-c[0])<r)&(np.abs(A[:,1]-c[1])<r)
Q = X[inpatch(X, 0.03)]
D = P[inpatch(P, 0.03+2*s)]
print(len(Q), len(D))
cs = s/3; csx = s/12
o = P.min(0) - cs
def cells(A):
    return np.floor((A[:,0]-o[0])/csx).astype(int), np.floor((A[:,1]-o[1])/cs).astype(int), np.floor((A[:,2]-o[2])/cs).astype(int)
dx_, dy_, dz_ = cells(D)
# sort D by (z,y,x)
from collections import defaultdict
rows = defaultdict(list)
for i,(a,b,cc) in enumerate(zip(dx_,dy_,dz_)): rows[(b,cc)].append(a)
rows = {k: np.sort(np.array(v)) for k,v in rows.items()}
T = cKDTree(D)
exact = np.array([len(T.query_ball_point(q, s)) for q in Q])
def chord_cells(q, yy, zz):
    y0 = o[1]+cs*yy; y1=y0+cs; z0=o[2]+cs*zz; z1=z0+cs
    gy = max(0, y0-q[1], q[1]-y1); gz = max(0, z0-q[2], q[2]-z1)
    rem = s*s-gy*gy-gz*gz
    if rem < 0: return None
    hx = np.sqrt(rem)
    return int(np.floor((q[0]-hx-o[0])/csx)), int(np.floor((q[0]+hx-o[0])/csx))
def count_rows(qs):
    # union of chords per row (min lo, max hi) -> count
    ys = np.floor((qs[:,1]-o[1])/cs).astype(int); zs = np.floor((qs[:,2]-o[2])/cs).astype(int)
    tot = 0; per = np.zeros(len(qs))
    for yy in range(ys.min()-3, ys.max()+4):
        for zz in range(zs.min()-3, zs.max()+4):
            r = rows.get((yy,zz))
            if r is None: continue
            lo=10**9; hi=-10**9
            for k,q in enumerate(qs):
                ch = chord_cells(q,yy,zz)
                if ch is None: continue
                lo=min(lo,ch[0]); hi=max(hi,ch[1])
                per[k] += np.searchsorted(r, ch[1], 'right') - np.searchsorted(r, ch[0], 'left')
            if lo<=hi: tot += np.searchsorted(r, hi, 'right') - np.searchsorted(r, lo, 'left')
    return tot, per
# Morton order of half-cells
def morton(q):
    h = np.floor((q - o)/(s/6)).astype(np.int64)
    code = np.zeros(len(q), np.int64)
    for b in range(10):
        for a in range(3):
            code |= ((h[:,a]>>b)&1) << (3*b+a)
    return code
order = np.argsort(morton(Q), kind='stable')
Qs = Q[order]; ex = exact[order]
G=int(sys.argv[1]) if len(sys.argv)>1 else 8
tot_union=0; tot_per=0; tot_max=0; tot_ex=0; ng=0
for g0 in range(0, len(Qs)-G+1, G):
    qs = Qs[g0:g0+G]
    t, per = count_rows(qs)
    tot_union += t*G; tot_per += per.sum(); tot_max += per.max()*G; tot_ex += ex[g0:g0+G].sum(); ng+=1
    if ng>=150: break
print(f"G={G} groups={ng}: union/exact {tot_union/tot_ex:.3f}  perquery/exact {tot_per/tot_ex:.3f}  maxper/exact {tot_max/tot_ex:.3f}")
# pairs inside groups of 8: pair-union row counts, max over the 4 pairs
tp=0; tmax=0; tex=0; ng=0
for g0 in range(0, len(Qs)-8+1, 8):
    us=[]
    for p in range(4):
        t,_ = count_rows(Qs[g0+2*p:g0+2*p+2]); us.append(t)
    tp += sum(us)*2; tmax += max(us)*8; tex += ex[g0:g0+8].sum(); ng+=1
    if ng>=100: break
print(f"pairs in groups of 8: pairunion/exact {tp/tex:.3f}  maxpair/exact {tmax/tex:.3f}")

import numpy as np
from scipy.spatial import cKDTree
rng=np.random.default_rng(1)
L=28.0; rho=0.75; n=int(rho*L**3)
x=rng.random((n,3))*L
a=2.8; nc=int(L//a); a=L/nc
c=np.floor(x/a).astype(int)%nc
# column order: cells ordered x,y column then z; in-cell random (entry id)
key=(c[:,0]*nc+c[:,1])*nc+c[:,2]
order=np.lexsort((np.arange(n),key))
R=2.6
tree=cKDTree(x,boxsize=L)
nb=[set(s)-{i} for i,s in enumerate(tree.query_ball_point(x,R))]
def ratio(pairs):
    tot=0;un=0
    for a_,b_ in pairs:
        A=nb[a_];B=nb[b_]
        tot+=len(A)+len(B); un+=len(A|B)
    return un/tot*2
# consecutive within column (approximate tiles by columns)
cons=[(order[i],order[i+1]) for i in range(0,n-1,2)]
print("consecutive union/n", ratio(cons[:20000]))
# MNN in chunks of 64
def mnn(ch,rounds=4):
    P=x[ch]; m=len(ch); d=np.linalg.norm(((P[:,None,:]-P[None,:,:])+L/2)%L-L/2,axis=2); np.fill_diagonal(d,1e9)
    match=-np.ones(m,int)
    for r in range(rounds):
        un=match<0
        dd=d.copy(); dd[:,~un]=1e9
        best=dd.argmin(1)
        for i in range(m):
            if un[i] and best[i]!=i and un[best[i]] and best[best[i]]==i: match[i]=best[i]
    left=[i for i in range(m) if match[i]<0]
    for k in range(0,len(left)-1,2): match[left[k]]=left[k+1]; match[left[k+1]]=left[k]
    return [(ch[i],ch[match[i]]) for i in range(m) if match[i]>i]
pr=[]
for s in range(0,min(n,20000)-64,64): pr+=mnn(order[s:s+64])
print("mnn union/n", ratio(pr))
dist=lambda p: np.mean([np.linalg.norm(((x[a_]-x[b_])+L/2)%L-L/2) for a_,b_ in p])
print("mean d cons", dist(cons[:10000]), "mnn", dist(pr))

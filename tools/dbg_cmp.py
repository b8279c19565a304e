import numpy as np, sys
a=np.load('/tmp/g5.npz'); b=np.load('/tmp/g2.npz')
g5,g2=a['g'],b['g']
R=int(sys.argv[1])
print('rhs', np.abs(a['r']-b['r']).max()/np.abs(b['r']).max())
d=np.abs(g5-g2); print('gram', d.max()/np.abs(g2).max())
G5=g5.reshape(R,R,R,R,R,R); G2=g2.reshape(R,R,R,R,R,R)
D=np.abs(G5-G2); thr=1e-9*np.abs(G2).max()
print('bad (p2,q2):', np.argwhere(D.max(axis=(0,2,3,5))>thr)[:20].tolist())
print('bad (p3,q3):', np.argwhere(D.max(axis=(0,1,3,4))>thr)[:20].tolist())
print('bad (p1,q1):', np.argwhere(D.max(axis=(1,2,4,5))>thr)[:20].tolist())

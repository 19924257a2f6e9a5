import numpy as np
E=np.load('gpurun_out/fwd_timeline_raw.npy').astype(np.float64)
c=np.nonzero((E>0).all(axis=0))[0]; c=c[c>16]
def pct(x): return f"p10 {np.percentile(x,10):6.0f} p50 {np.percentile(x,50):6.0f} p90 {np.percentile(x,90):6.0f}"
k=c[np.isin(c-2,c)]
print('producer reached chunk -> vmeta acquired:', pct(E[5][c]-E[4][c]))
print('vmeta acquired -> K issued (kempty wait):', pct(E[0][c]-E[5][c]))
print('K(k-1) issued -> producer reached k:', pct(E[4][k]-E[0][k-1]))
print('S(k-2) issued -> producer reached k:', pct(E[4][k]-E[2][k-2]))
print('K(k) issued - S(k-2) issued:', pct(E[0][k]-E[2][k-2]))

import numpy as np, sys
d=np.load('gpurun_out/trace_c3_plain.npz')
st=d['st']; tk=d['tk']; nf=int(d['nf'])
sup=np.load(sys.argv[1]) if len(sys.argv)>1 else None
GHZ=1.965
f=st[:nf].astype(np.float64); t=tk[:nf]
R=t[:,2]-t[:,1]
own=(f[:,7]-f[:,4])/GHZ/1e3; bar=(f[:,8]-f[:,7])/GHZ/1e3; epi=(f[:,5]-f[:,8])/GHZ/1e3
for lo,hi in [(1,8),(8,16),(16,32),(32,64),(64,128),(128,257)]:
    m=(R>=lo)&(R<hi)
    if m.sum(): print(f"R in [{lo},{hi}): {m.sum()} tasks  own matvec {own[m].mean():.2f}  barrier {bar[m].mean():.2f}  epilogue {epi[m].mean():.2f} us; rg {t[m,3].mean():.1f}")

"""Third-order (KdV-type) equations in the oracle with literal (h^k) and unit-scaled derivative rows:
relative u_phi error against u_t + u_xxx = f (forced) and the Airy wave u = sin(pi x + pi^3 t)
at n = 16, 32, 64 (reading O3).  CPU; calls only oracle/."""
import numpy as np, sys, scipy.sparse as sp
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import oracle.neurlp as nl
from oracle import Problem, assemble
def solve(pr, c, b, om, unit):
    A,d,info=assemble(pr,c,b,om)
    if unit:
        P=pr.P; r0=P+info['bnd_rows'].size
        sc=np.ones(A.shape[0])
        for dd in range(pr.D):
            for kk in range(1,pr.ord(dd)+1):
                sc[r0:r0+P]=1.0/pr.h[dd]**kk; r0+=P
        A=sp.diags(sc)@A; d=sc*d
    return nl.solve_normal(A, A.T@d, method='lu')
for case in ('forced','wave'):
  for unit in (False, True):
    errs=[]
    for n in (16,32,64):
        h=1.0/(n-1); ht = h if case=='forced' else 0.2*h
        pr=Problem((n,n),(ht,h),order=(2,3))
        t,x=np.meshgrid(np.arange(n)*ht, np.arange(n)*h, indexing='ij')
        k=np.pi
        c=np.zeros((pr.M,pr.P)); c[pr.field(1,3)]=1.0; c[pr.field(0,1)]=1.0
        if case=='forced':
            u=np.sin(k*x)*np.exp(-t); b=(-k**3*np.cos(k*x)*np.exp(-t) - np.sin(k*x)*np.exp(-t)).reshape(-1)
        else:
            u=np.sin(k*x+k**3*t); b=np.zeros(pr.P)
        z=solve(pr,c,b,u.reshape(-1),unit)
        errs.append(np.linalg.norm(z[:pr.P]-u.reshape(-1))/np.linalg.norm(u))
    print(case, 'unit' if unit else 'literal', ['%.2e'%e for e in errs])

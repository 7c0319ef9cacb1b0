"""numpy model of the one-sided Jacobi sweep count on the C2 Lanczos B_k
(scripts/B384_lanczos.npy, d = 384): (1) all-pairs circle ordering on B,
B^T, R / R^T of a (pivoted) QR of B (Drmac-style preconditioning); (2) the
device kernel's cyclic-by-blocks ordering with JC-column blocks, one pass of
JC cross rotations per round (the kernel) vs the block pair diagonalised
fully per round.  Development evidence for DESIGN.md section 6 (Jacobi).
Printed (round 2): B 14, B^T 12, R 14, R^T 10, R(no piv)^T 12, QRCP2 9;
JC=4 kernel 12 / full pair 13; JC=8 kernel 13 / full pair 12."""
import numpy as np, scipy.linalg as sl, sys, time
import os
B = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'B384_lanczos.npy'))
d = B.shape[0]
def sweeps(G, tol=None, maxs=40):
    G = G.copy(); n = G.shape[1]
    tol = tol or n * 2.0**-53
    nrm2 = (G*G).sum(0)
    for sw in range(maxs):
        rot = 0
        # round-robin (circle) ordering, all pairs per sweep; vectorised per round
        cols = list(range(n)) + ([n] if n % 2 else [])
        m = len(cols)
        for r in range(m - 1):
            ps = []; qs = []
            for t in range(m // 2):
                p = cols[t]; q = cols[m - 1 - t]
                if p < n and q < n: ps.append(p); qs.append(q)
            ps = np.array(ps); qs = np.array(qs)
            X = G[:, ps]; Y = G[:, qs]
            a = (X*X).sum(0); b = (Y*Y).sum(0); c = (X*Y).sum(0)
            do = np.abs(c) > tol*np.sqrt(a*b)
            rot += do.sum()
            h = 0.5*(b-a)
            t = np.where(do, np.sign(np.where(h>=0,1,-1))*c/(np.abs(h)+np.sqrt(h*h+c*c)), 0.0)
            cs = 1/np.sqrt(1+t*t); sn = cs*t
            G[:, ps] = cs*X - sn*Y; G[:, qs] = sn*X + cs*Y
            cols = [cols[0]] + [cols[-1]] + cols[1:-1]
        if rot == 0: return sw
    return maxs
s_ref = np.linalg.svd(B, compute_uv=False)
for name, M in [('B', B), ('B^T', B.T)]:
    t=time.time(); print(name, sweeps(M), f'{time.time()-t:.1f}s', flush=True)
Q, R, piv = sl.qr(B, pivoting=True)
print('R', sweeps(R), flush=True)
print('R^T', sweeps(R.T), flush=True)
Q2, R2 = np.linalg.qr(B)
print('R (no piv)^T', sweeps(R2.T), flush=True)
# two-step: QRCP then LQ of R -> L, Jacobi on L^T?  (Drmac: R^T then)
Q3, R3, p3 = sl.qr(R.T, pivoting=True)
print('R2 of QRCP(R^T) ^T', sweeps(R3.T), flush=True)

# --- (2) cyclic-by-blocks ordering ---
U = 2.0**-53; tol = d*U
def rot(G, p, q, absmin):
    x, y = G[:, p], G[:, q]
    a, b, c = x@x, y@y, x@y
    if not (a > absmin and b > absmin and c*c > tol*tol*a*b): return 0
    h = 0.5*(b-a); t = (c if h >= 0 else -c)/(abs(h)+np.sqrt(h*h+c*c))
    cs = 1/np.sqrt(1+t*t); sn = cs*t
    G[:, p], G[:, q] = cs*x - sn*y, sn*x + cs*y
    return 1
def circle(t, r, ne):
    p = 0 if t == 0 else ((t-1+r) % (ne-1))+1
    q = ((ne-2-t+r) % (ne-1))+1
    return min(p,q), max(p,q)
def run(JC, full_pair, maxs=40):
    nb = d//JC; G = B.copy(); absmin = (U*np.linalg.norm(B))**2
    for sw in range(maxs):
        nrot = 0
        for rnd in range(nb):
            for k in range(nb//2):
                if rnd == 0: bi, bj = 2*k, 2*k+1
                else: bi, bj = circle(k, rnd-1, nb)
                cols = list(range(bi*JC, bi*JC+JC)) + list(range(bj*JC, bj*JC+JC))
                if full_pair:
                    for inner in range(30):
                        r_in = 0
                        for i in range(2*JC):
                            for j in range(i+1, 2*JC): r_in += rot(G, cols[i], cols[j], absmin)
                        nrot += r_in
                        if r_in == 0: break
                else:
                    if rnd == 0:
                        for ir in range(JC-1):
                            h = JC//2
                            for t in range(JC):
                                off = 0 if t < h else JC; tt = t if t < h else t-h
                                p, q = circle(tt, ir, JC); nrot += rot(G, cols[off+p], cols[off+q], absmin)
                    else:
                        for ir in range(JC):
                            for t in range(JC): nrot += rot(G, cols[t], cols[JC+(t+ir) % JC], absmin)
        if nrot == 0: return sw
    return maxs
for JC in (4, 8):
    for fp in (False, True):
        t = time.time(); print(JC, fp, run(JC, fp), f'{time.time()-t:.0f}s', flush=True)

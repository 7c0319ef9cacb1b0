"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds ONLY input generation: prescribed spectra, dense test
matrices A = X.Sigma.Y^T and CSR matrices with power-law row/column lengths.
It contains none of the method's arithmetic (no products with A, no
orthogonalisation, no SVD of the projected matrix).  The random numbers the
*method* draws (start blocks, breakdown replacements) are NOT produced here:
each side implements the same counter-based Philox generator (oracle/philox.py
and csrc/philox.cuh).

Recipes:
  * spectrum_eq16  - Eq. 16 (Sec. 4.2), read as the SET
    {10^(30 i/n - 14)}, i = 1..n/2, plus n/2 copies of 1e-14, sorted
    descending.
  * dense_prescribed - Eq. 15: A = X Sigma Y^T with X, Y
    orthogonal.  Small sizes: X, Y = Householder Q of a Gaussian matrix.
    Large sizes: products of `n_reflectors` random Householder reflectors
    (O(mn) to form, exact spectrum).
  * powerlaw_csr (G1, Chung-Lu) - row lengths from a Pareto tail with
    exponent alpha (density ~ x^-alpha), columns drawn from Pareto weights
    under a random permutation, duplicates summed, values N(0,1).  Shapes of
    the paper's SuiteSparse set (Table 2).
  * blockdiag_csr (G2) - A = Pi_r blockdiag(B_1..B_T) Pi_c^T with dense
    blocks of prescribed spectra, so sigma(A) = union sigma(B_t) exactly.
"""
from __future__ import annotations

import os

import numpy as np

__all__ = [
    "spectrum_eq16",
    "dense_prescribed",
    "powerlaw_csr",
    "powerlaw_csr_device",
    "blockdiag_csr",
    "gaussian_block",
    "CONFIGS",
    "SEEDS",
]

SEEDS = {
    "C1": 0x2403062181,
    "C2": 0x2403062182,
    "C3": 0x2403062183,
    "C4": 0x2403062184,
    "C5": 0x2403062185,
    "C5s": 0x2403062185,
    "C5g2": 0x2403062186,
}

# BASELINE.json configs with the solver settings of SURVEY.md 8(a)/8(d).
CONFIGS = {
    "C1": dict(kind="dense", m=200, n=100, r=10, b=4, d=28, tol=1e-12, maxit=8,
               rsvd_p=10, rsvd_q=1),
    "C2": dict(kind="csr", m=1_000_000, n=1_000_000, nnz=10_000_000, alpha=2.5,
               r=50, b=16, d=384, tol=1e-8, maxit=6),
    "C3": dict(kind="csr", m=4_000_000, n=500_000, nnz=50_000_000, alpha=2.5,
               r=100, b=32, d=640, tol=1e-8, maxit=6, rsvd_p=10, rsvd_q=2),
    "C4": dict(kind="dense", m=40_000, n=20_000, r=200, b=32, d=704, tol=1e-6,
               maxit=6, rsvd_p=10, rsvd_q=8),
    # C5 (i): fixed-work runs, one restart cycle at d = 160; the
    # matrix is generated on the device (powerlaw_csr_device)
    "C5": dict(kind="csr", m=50_000_000, n=50_000_000, nnz=1_000_000_000,
               alpha=2.5, r=100, b=32, d=160, tol=1e-8, maxit=1, device_gen=True),
    # C5 (iii): the G2 twin at C5 scale (blockdiag_csr_device: closed-form
    # spectrum, top 100 = linspace(200, 100), tail <= 20; mean row ~20 ->
    # nnz ~1e9), LancSVD to tol with thick restart (keep 128) on one GPU
    "C5g2": dict(kind="csr", m=50_000_000, n=50_000_000, nnz=1_000_000_000, alpha=2.5,
                 mean_block=2.6, top=(200.0, 100.0, 100), tail_max=20.0,
                 r=100, b=32, d=160, keep=128, tol=1e-8, maxit=40, device_gen="g2"),
    # C5 scaled down by 10 (SURVEY 8(d) "Oracle timing"): the host oracle's sample
    "C5s": dict(kind="csr", m=5_000_000, n=5_000_000, nnz=100_000_000,
                alpha=2.5, r=100, b=32, d=160, tol=1e-8, maxit=1),
}


def spectrum_eq16(n: int) -> np.ndarray:
    """Eq. 16, set reading: sigma_i =
    10^(1 - 30(i-1)/n) for i <= n/2, else 1e-14; descending."""
    i = np.arange(1, n + 1, dtype=np.float64)
    s = np.where(i <= n // 2, 10.0 ** (1.0 - 30.0 * (i - 1.0) / n), 1e-14)
    return np.sort(s)[::-1].copy()


def gaussian_block(rows: int, cols: int, seed: int) -> np.ndarray:
    """Input-side Gaussian (PCG64), for test operands only - never a start
    block of the method."""
    return np.random.default_rng(seed).standard_normal((rows, cols))


def _householder_q(rows: int, cols: int, rng) -> np.ndarray:
    g = rng.standard_normal((rows, cols))
    q, r = np.linalg.qr(g)
    return q * np.sign(np.diag(r))


def dense_prescribed(m: int, n: int, sigma: np.ndarray, seed: int,
                     n_reflectors: int | None = None, xp="numpy", device=None):
    """A = X diag(sigma) Y^T (Eq. 15), row-major float64 m x n.

    n_reflectors=None: X (m x n), Y (n x n) dense random orthogonal (small m, n).
    n_reflectors=k: X = H_1..H_k [I;0], Y = G_1..G_k with random unit
    reflectors; cost O(k m n).  xp="torch" builds it with torch on `device`
    (same recipe, rounding may differ from numpy in the last bits; the oracle
    is always handed the bytes actually used)."""
    sigma = np.asarray(sigma, dtype=np.float64)
    assert m >= n and sigma.shape == (n,)
    rng = np.random.default_rng(seed)
    if n_reflectors is None:
        X = _householder_q(m, n, rng)
        Y = _householder_q(n, n, rng)
        A = (X * sigma[None, :]) @ Y.T
        if xp == "torch":
            import torch
            return torch.from_numpy(np.ascontiguousarray(A)).to(device)
        return np.ascontiguousarray(A)
    xs = [rng.standard_normal(m) for _ in range(n_reflectors)]
    ys = [rng.standard_normal(n) for _ in range(n_reflectors)]
    xs = [x / np.linalg.norm(x) for x in xs]
    ys = [y / np.linalg.norm(y) for y in ys]
    if xp == "torch":
        import torch
        A = torch.zeros((m, n), dtype=torch.float64, device=device)
        A.diagonal().copy_(torch.from_numpy(sigma))
        # rank-1 updates in place (addr_): no m x n temporaries, so m = 1e6,
        # n = 1e4 (80 GB) builds within the device memory
        for y in ys:  # A <- A (I - 2 y y^T)   (Y^T from the right)
            yt = torch.from_numpy(y).to(device)
            A.addr_(A @ yt, yt, alpha=-2.0)
        for x in xs:  # A <- (I - 2 x x^T) A
            xt = torch.from_numpy(x).to(device)
            A.addr_(xt, xt @ A, alpha=-2.0)
        return A
    A = np.zeros((m, n))
    A[np.arange(n), np.arange(n)] = sigma
    for y in ys:
        A -= 2.0 * np.outer(A @ y, y)
    for x in xs:
        A -= 2.0 * np.outer(x, x @ A)
    return A


def _pareto_weights(k: int, alpha: float, rng) -> np.ndarray:
    # density ~ x^-alpha on [1, inf)  <=>  tail P(X > x) = x^-(alpha-1)
    u = rng.random(k)
    return (1.0 - u) ** (-1.0 / (alpha - 1.0))


def _row_lengths(m: int, n: int, nnz: int, alpha: float, rng) -> np.ndarray:
    w = _pareto_weights(m, alpha, rng)
    target = w * (nnz / w.sum())
    target = np.minimum(target, n)
    L = np.floor(target).astype(np.int64)
    rem = int(nnz - L.sum())
    if rem > 0:
        frac = target - L
        frac[L >= n] = -1.0
        idx = np.argpartition(-frac, min(rem, m - 1))[:rem]
        L[idx] += 1
    return np.minimum(L, n)


def powerlaw_csr(m: int, n: int, nnz: int, alpha: float, seed: int,
                 exact_after_dedup: bool = True):
    """G1 Chung-Lu CSR: returns (rowptr int64[m+1],
    colidx int32[nnz'], vals f64[nnz']) canonical (sorted, duplicates summed).
    Duplicates are summed, which loses entries; with exact_after_dedup the
    draw is repeated once with the draw count scaled by the observed loss so
    nnz' is within ~1% of nnz."""
    out = _powerlaw_csr(m, n, nnz, alpha, seed, 1.0)
    if exact_after_dedup and len(out[1]) < 0.99 * nnz:
        out = _powerlaw_csr(m, n, nnz, alpha, seed, nnz / max(1, len(out[1])))
    return out


def _powerlaw_csr(m, n, nnz, alpha, seed, oversample):
    rng = np.random.default_rng(seed)
    L = _row_lengths(m, n, int(nnz * oversample), alpha, rng)
    cw = _pareto_weights(n, alpha, rng)
    cw = cw[rng.permutation(n)]
    cdf = np.cumsum(cw)
    cdf /= cdf[-1]
    total = int(L.sum())
    rows = np.repeat(np.arange(m, dtype=np.int64), L)
    cols = np.searchsorted(cdf, rng.random(total), side="right").astype(np.int64)
    np.minimum(cols, n - 1, out=cols)
    vals = rng.standard_normal(total)
    key = rows * n + cols
    order = np.argsort(key, kind="stable")
    key = key[order]
    vals = vals[order]
    uniq, start = np.unique(key, return_index=True)
    vsum = np.add.reduceat(vals, start) if len(start) else vals[:0]
    r = (uniq // n).astype(np.int64)
    c = (uniq % n).astype(np.int32)
    rowptr = np.zeros(m + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(np.bincount(r, minlength=m))
    return rowptr, c, np.ascontiguousarray(vsum, dtype=np.float64)


def powerlaw_csr_device(m: int, n: int, nnz: int, alpha: float, seed: int, device="cuda",
                        exact_after_dedup: bool = True):
    """G1 Chung-Lu CSR generated with torch on `device` -- the same recipe
    and distributions as powerlaw_csr, for C5 (m = n = 5e7, nnz = 1e9), where
    the host generator would need many minutes and > 60 GB of host memory.
    The random stream is torch's (Philox on CUDA), so the bytes differ from
    powerlaw_csr at the same seed; they are deterministic for a given seed and
    device type.  Returns (rowptr int64[m+1], colidx int32, vals f64) tensors
    on `device`, canonical (sorted, duplicates summed in sorted order)."""
    out = _powerlaw_csr_device(m, n, nnz, alpha, seed, 1.0, device)
    if exact_after_dedup and out[1].numel() < 0.99 * nnz:
        got = out[1].numel()
        del out
        out = _powerlaw_csr_device(m, n, nnz, alpha, seed, nnz / max(1, got), device)
    return out


def _powerlaw_csr_device(m, n, nnz, alpha, seed, oversample, device):
    import sys
    import time
    import torch
    t0 = time.time()

    def log(what):
        if os.environ.get("TSVD_GEN_VERBOSE"):
            print(f"[gen] {what}: {time.time() - t0:.1f} s", file=sys.stderr, flush=True)
    f64 = torch.float64
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    want = int(nnz * oversample)
    # row lengths (_row_lengths): Pareto weights scaled to the mean, capped at n
    u = torch.rand(m, generator=g, dtype=f64, device=device)
    target = (1.0 - u) ** (-1.0 / (alpha - 1.0))
    target = torch.clamp(target * (want / float(target.sum())), max=float(n))
    L = torch.floor(target).to(torch.int64)
    rem = want - int(L.sum())
    if rem > 0:
        frac = target - L
        frac[L >= n] = -1.0
        idx = torch.argsort(frac, descending=True)[:min(rem, m)]
        L[idx] += 1
        del frac, idx
    L.clamp_(max=n)
    del u, target
    log("row lengths")
    # column weights under a random permutation, inverse-CDF draws
    u = torch.rand(n, generator=g, dtype=f64, device=device)
    cw = ((1.0 - u) ** (-1.0 / (alpha - 1.0)))[torch.randperm(n, generator=g, device=device)]
    cdf = torch.cumsum(cw, 0)
    cdf /= cdf[-1].clone()
    del u, cw
    total = int(L.sum())
    key = torch.repeat_interleave(torch.arange(m, device=device, dtype=torch.int64), L)
    key *= n
    cols = torch.searchsorted(cdf, torch.rand(total, generator=g, dtype=f64, device=device),
                              right=True)
    cols.clamp_(max=n - 1)
    key += cols
    del cols, cdf, L
    log("keys")
    vals = torch.randn(total, generator=g, dtype=f64, device=device)
    key, order = torch.sort(key, stable=True)
    vals = vals[order]
    del order
    log("sort")
    uniq, counts = torch.unique_consecutive(key, return_counts=True)
    del key
    if uniq.numel() < total:
        vals = torch.segment_reduce(vals, "sum", lengths=counts)
    del counts
    r = uniq // n
    colidx = (uniq - r * n).to(torch.int32)
    del uniq
    rowptr = torch.zeros(m + 1, dtype=torch.int64, device=device)
    rowptr[1:] = torch.cumsum(torch.bincount(r, minlength=m), 0)
    del r
    log("dedup + rowptr")
    return rowptr, colidx, vals.contiguous()


def blockdiag_csr(m: int, n: int, mean_row: float, alpha: float, seed: int,
                  top_sigma: np.ndarray, tail_max: float = 1.0,
                  max_width: int = 256):
    """G2: A = Pi_r blockdiag(B_1..B_T) Pi_c^T.  Block widths
    n_t follow a Pareto tail (power-law row lengths, row length = n_t); block
    heights m_t = n_t * (m/n) rounded.  Each B_t = X_t diag(s_t) Y_t^T.
    The len(top_sigma) largest singular values are `top_sigma` (assigned to
    random blocks); every other value is uniform in (0, tail_max).
    Returns (rowptr, colidx, vals, sigma_all_sorted_desc)."""
    rng = np.random.default_rng(seed)
    top_sigma = np.sort(np.asarray(top_sigma, dtype=np.float64))[::-1]
    aspect = m / n
    widths = []
    total_n = 0
    while total_n < n:
        w = int(min(max_width, max(1, round(_pareto_weights(1, alpha, rng)[0]
                                              * mean_row * (alpha - 2.0) / (alpha - 1.0)))))
        w = min(w, n - total_n)
        widths.append(w)
        total_n += w
    widths = np.array(widths, dtype=np.int64)
    heights = np.maximum(widths, np.round(widths * aspect).astype(np.int64))
    # fix the total height to m (adjust from the back, keep m_t >= n_t)
    excess = int(heights.sum() - m)
    t = len(heights) - 1
    while excess != 0 and t >= 0:
        if excess > 0:
            dec = min(excess, int(heights[t] - widths[t]))
            heights[t] -= dec
            excess -= dec
        else:
            heights[t] += -excess
            excess = 0
        t -= 1
    if excess > 0:
        raise ValueError("cannot fit blocks into m rows; lower mean_row")
    T = len(widths)
    nsig = int(widths.sum())
    sig = rng.random(nsig) * tail_max
    k = len(top_sigma)
    pos = rng.choice(nsig, size=k, replace=False)
    sig[pos] = top_sigma
    sig_off = np.concatenate([[0], np.cumsum(widths)])
    rperm = rng.permutation(m)
    cperm = rng.permutation(n)
    row_off = np.concatenate([[0], np.cumsum(heights)])
    rows_l, cols_l, vals_l = [], [], []
    for t in range(T):
        mt, nt = int(heights[t]), int(widths[t])
        s = sig[sig_off[t]:sig_off[t + 1]]
        X = _householder_q(mt, nt, rng)
        Y = _householder_q(nt, nt, rng)
        B = (X * s[None, :]) @ Y.T
        gr = rperm[row_off[t]:row_off[t + 1]]
        gc = cperm[sig_off[t]:sig_off[t + 1]]
        rows_l.append(np.repeat(gr, nt))
        cols_l.append(np.tile(gc, mt))
        vals_l.append(B.ravel())
    rows = np.concatenate(rows_l).astype(np.int64)
    cols = np.concatenate(cols_l).astype(np.int64)
    vals = np.concatenate(vals_l)
    order = np.argsort(rows * n + cols, kind="stable")
    rows, cols, vals = rows[order], cols[order], vals[order]
    rowptr = np.zeros(m + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(np.bincount(rows, minlength=m))
    sigma_all = np.sort(np.concatenate([sig, np.zeros(max(0, n - nsig))]))[::-1]
    return rowptr, cols.astype(np.int32), np.ascontiguousarray(vals), sigma_all


def blockdiag_csr_device(m: int, n: int, mean_row: float, alpha: float, seed: int,
                         top_sigma, tail_max: float = 1.0, max_width: int = 256,
                         device="cuda", chunk_rows: int = 4_000_000):
    """G2 at C5 scale, generated with torch on `device`:
    A = Pi_r blockdiag(B_1..B_T) Pi_c^T, square blocks (m = n), widths n_t
    from the same Pareto recipe as blockdiag_csr (row length = n_t: power-law
    rows), B_t = H(x_t) diag(s_t) H(y_t) with Householder reflectors
    H(v) = I - 2 v v^T (unit v), so sigma(B_t) = s_t exactly and
    sigma(A) = union of the s_t (closed form).  The len(top_sigma) largest
    values are `top_sigma` (placed in random blocks), every other one is
    uniform in (0, tail_max).  Entry (i, j) of B_t, written out:
        s_i [i == j] - 2 x_i x_j s_j - 2 s_i y_i y_j + 4 c_t x_i y_j,
        c_t = sum_k x_k s_k y_k.
    The columns a block owns are a random subset of [0, n) in increasing
    order (so every CSR row comes out sorted: canonical without a sort of
    the nonzeros).  Returns (rowptr int64[m+1], colidx int32, vals f64,
    sigma_all_sorted_desc as a numpy array); O(nnz) work, rows generated in
    chunks to bound the temporaries."""
    import torch
    if m != n:
        raise ValueError("blockdiag_csr_device builds square blocks (m = n)")
    f64, i64 = torch.float64, torch.int64
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    scale = mean_row * (alpha - 2.0) / (alpha - 1.0)
    # block widths: Pareto draws, rounded, capped; cut where the sum reaches n
    est = int(2.5 * n / max(1.0, mean_row)) + 1024
    u = torch.rand(est, generator=g, dtype=f64, device=device)
    w = torch.clamp(torch.round((1.0 - u) ** (-1.0 / (alpha - 1.0)) * scale), 1, max_width).to(i64)
    csum = torch.cumsum(w, 0)
    T = int(torch.searchsorted(csum, torch.tensor([n], device=device, dtype=i64)).item()) + 1
    w = w[:T].clone()
    w[-1] -= int(csum[T - 1].item()) - n          # the last block ends exactly at n
    start = torch.zeros(T + 1, dtype=i64, device=device)
    start[1:] = torch.cumsum(w, 0)
    del u, csum
    # per column slot: its block, the singular value, the reflector vectors
    blk = torch.repeat_interleave(torch.arange(T, device=device, dtype=i64), w)
    s = torch.rand(n, generator=g, dtype=f64, device=device) * tail_max
    top = torch.as_tensor(np.sort(np.asarray(top_sigma, dtype=np.float64))[::-1].copy(),
                          device=device)
    pos = torch.randperm(n, generator=g, device=device)[:top.numel()]
    s[pos] = top
    x = torch.randn(n, generator=g, dtype=f64, device=device)
    y = torch.randn(n, generator=g, dtype=f64, device=device)
    for v in (x, y):
        nrm = torch.zeros(T, dtype=f64, device=device).index_add_(0, blk, v * v)
        v /= torch.sqrt(nrm)[blk]
    cblk = torch.zeros(T, dtype=f64, device=device).index_add_(0, blk, x * s * y)
    # rows: global row g <- slot rinv[g]; columns: block t owns a random
    # subset of [0, n), sorted, at slots start[t] .. start[t+1]-1
    rinv = torch.randperm(n, generator=g, device=device)
    cp = torch.randperm(n, generator=g, device=device)
    key = blk * n + cp
    cols_sorted = (torch.sort(key).values - blk * n).to(torch.int32)
    del key, cp
    L = w[blk[rinv]]                              # row lengths in global row order
    rowptr = torch.zeros(m + 1, dtype=i64, device=device)
    rowptr[1:] = torch.cumsum(L, 0)
    nnz = int(rowptr[-1].item())
    colidx = torch.empty(nnz, dtype=torch.int32, device=device)
    vals = torch.empty(nnz, dtype=f64, device=device)
    for r0 in range(0, m, chunk_rows):
        r1 = min(m, r0 + chunk_rows)
        z0, z1 = int(rowptr[r0].item()), int(rowptr[r1].item())
        grow = torch.repeat_interleave(torch.arange(r0, r1, device=device, dtype=i64),
                                       L[r0:r1])
        j = torch.arange(z0, z1, device=device, dtype=i64) - rowptr[grow]
        slot_i = rinv[grow]                       # row slot (local i = slot_i - start[t])
        t = blk[slot_i]
        slot_j = start[t] + j                     # column slot of local column j
        xi, yi, si = x[slot_i], y[slot_i], s[slot_i]
        xj, yj, sj = x[slot_j], y[slot_j], s[slot_j]
        v = -2.0 * xi * xj * sj - 2.0 * si * yi * yj + 4.0 * cblk[t] * xi * yj
        v += torch.where(slot_i == slot_j, si, torch.zeros_like(si))
        colidx[z0:z1] = cols_sorted[slot_j]
        vals[z0:z1] = v
        del grow, j, slot_i, t, slot_j, xi, yi, si, xj, yj, sj, v
    sigma_all = np.sort(s.cpu().numpy())[::-1]
    return rowptr, colidx, vals, sigma_all

"""CPU oracle for the truncated-SVD hot path of Tomas, Quintana-Orti, Anzt,
"Fast Truncated SVD of Sparse and Dense Matrices on Graphics Processors"
(arXiv 2403.06218; /root/reference/PAPER.md, cited as P:<line>).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py may import anything under
oracle/.  The product path (paper_2403_06218_b200/) never imports it and has
no CPU fallback.

Plain, slow, obviously correct numpy/scipy in IEEE float64.  Each
function follows the paper's algorithm step by step, with the readings listed
in DESIGN.md ("Readings of the paper") where the printed text is wrong or
silent.  Library primitives used as single steps: dense matmul (numpy),
CSR matmul (scipy.sparse), Cholesky (LAPACK potrf via numpy), triangular
solve (scipy), small SVD (LAPACK gesvd via scipy, exactly the paper's
choice, Table 1).

Pins (tests/test_oracle_*.py, -m "not gpu"): Philox KAT vectors, Householder
QR, closed-form spectra (Eq. 15/16), algebraic identities (Eq. 4-12), special
cases (d = n, l = n, b = 1, diagonal A, rank-deficient A), Eckart-Young.
Every function exported here has pins.  What the GPU parity tests compare
is the part of a result that is unique: converged triplets (sigma, residuals,
and singular vectors after the sign rule where sigma is separated), every
factor of the orthogonalisations, every kernel output.  Two things are not
unique across summation orders (reading R29) and are checked for validity
instead of equality: the iterate of triplets that have NOT converged (both
sides must still satisfy the Lanczos relations, orthonormal bases, and rho
consistent with the explicit residual), and the CGS2 branch decision for a
Cholesky pivot lying exactly at the breakdown threshold (the tests drive the
branch with exactly-zero pivots, where both sides must take it).
"""
from .philox import gaussian_block, philox4x32_10  # noqa: F401
from .core import (  # noqa: F401
    Operator, DrawCtx, chol, trsm_right_lt, cholqr2, cgs_cqr2, bcgs_pip2, cgs2, cgs_qr,
    small_svd, sign_normalize,
)
from .lancsvd import lancsvd, lancsvd_threshold  # noqa: F401
from .randsvd import randsvd  # noqa: F401
from .residual import residuals, eckart_young_2norm  # noqa: F401

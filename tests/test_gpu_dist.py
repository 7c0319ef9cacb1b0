"""The multi-GPU (row-partitioned, NCCL) code path on one GPU (-m gpu).

The driver's GPU tier has a single B200, so the NCCL path runs with world = 1
(handles created through tsvd_create_*_dist always run the reduce-scatter /
all-gather / all-reduce collectives); its result must equal the single-GPU
path.  The decomposition for world > 1 is checked on CPU with gloo
(tests/test_dist_gloo.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2403_06218_b200 as T  # noqa: E402
from tsvd_inputs import SEEDS, dense_prescribed, powerlaw_csr, spectrum_eq16  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _dist(m, n):
    return dict(rank=0, world=1, nccl_id=T.nccl_unique_id(), m_global=m, n_global=n,
                row_begin=0, row_end=m)


def _solve(h, algo):
    h.set_seed(5)
    if algo == "lanczos":
        st = h.block_lanczos(r=10, b=4, tol=1e-10, maxit=6, d=40)
    elif algo == "thick":
        h.set_thick_restart(16)
        st = h.block_lanczos(r=10, b=4, tol=1e-10, maxit=6, d=28)
    else:
        st = h.rsvd(r=10, p=6, q=2)
    return st, h.get()


@pytest.mark.parametrize("algo", ["lanczos", "rsvd", "thick"])
@pytest.mark.parametrize("kind", ["dense", "csr"])
def test_dist_world1_equals_single(kind, algo):
    if kind == "dense":
        A = dense_prescribed(300, 120, spectrum_eq16(120), SEEDS["C1"])
        m, n = A.shape
        kw = dict(A=A)
    else:
        m, n = 6000, 4000
        csr = powerlaw_csr(m, n, 60000, 2.5, seed=9)
        kw = dict(csr=csr, shape=(m, n))
    with T.TruncatedSVD(**kw) as h:
        st1, (U1, S1, V1) = _solve(h, algo)
    kw2 = dict(kw)
    kw2.pop("shape", None)
    with T.TruncatedSVD(**kw2, dist=_dist(m, n)) as h:
        st2, (U2, S2, V2) = _solve(h, algo)
        info = h.info()
    assert st1 == st2
    assert info["launches"] > 0
    assert np.abs(S1 - S2).max() <= 1e-14 * S1[0]
    assert np.abs(U1 - U2).max() <= 1e-12 and np.abs(V1 - V2).max() <= 1e-12

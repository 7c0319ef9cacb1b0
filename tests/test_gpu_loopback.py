"""The library's row-partitioned multi-GPU code path at world > 1 (-m gpu).

One GPU only, so the ranks are `world` handles on the same device, one host
thread each, joined by the library's test-only loopback communicator
(tsvd_loopback_create: the collectives go through device memory instead of
NCCL, rank-ordered sums).  Everything else is the code a multi-GPU run
executes: nnz-balanced row shards of A, local CSR(A_g^T),
n-shards of P padded to ceil(n / world), the reduce-scatter of A_g^T Qbar,
the all-gather of Q_i before A_g Q_i, all-reduced projections and Grams,
Philox draws by GLOBAL row (start block, CGS2 replacement columns), the
gathered sign rule, replicated B_k / Jacobi / rho / restart decisions, and
the all-reduced explicit residuals.

The result must equal the single-GPU handle's up to the summation order of
the row-sharded reductions, on the triplets converged in the single run
(north_star: acceptance is over converged triplets; an unconverged Ritz
pair is defined by the iteration and moves with the rounding path): sigma
to 1e-12 sigma_1, vectors (sign rule applied on both) to 1e-9, same cycle
count and status.  Covers world 2 and 3, sparse
and dense A, LancSVD (paper restart and thick restart) and RandSVD, and a
rank whose row range AND n-shard are empty (the zero Gram
partial of an empty shard)."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_2403_06218_b200 as T  # noqa: E402
from tsvd_inputs import SEEDS, dense_prescribed, powerlaw_csr, spectrum_eq16  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _solve(h, algo):
    h.set_seed(5)
    if algo == "pip2":   # the single-reduction orthogonalisation
        h.set_ortho("bcgs_pip2")
        algo = "lanczos"
    if algo == "lanczos":
        st = h.block_lanczos(r=10, b=4, tol=1e-10, maxit=6, d=40)
    elif algo == "thick":
        h.set_thick_restart(16)
        st = h.block_lanczos(r=10, b=4, tol=1e-10, maxit=6, d=28)
    else:
        st = h.rsvd(r=10, p=6, q=2)
    U, S, V = h.get()
    e, _ = h.residuals()
    conv = h.rho() <= 1e-10 if algo != "rsvd" else e <= 1e-10
    return st, U, S, V, e, h.info(), conv


def _run_world(kind, data, m, n, bounds, algo):
    world = len(bounds) - 1
    grp = T.LoopbackGroup(world)
    out = [None] * world
    err = []

    def rank_main(g):
        try:
            torch.cuda.set_device(0)
            r0, r1 = int(bounds[g]), int(bounds[g + 1])
            dist = dict(rank=g, world=world, nccl_id=None, loopback=grp, m_global=m,
                        n_global=n, row_begin=r0, row_end=r1)
            if kind == "dense":
                kw = dict(A=np.ascontiguousarray(data[r0:r1]))
            else:
                rp, ci, va = data
                lo, hi = int(rp[r0]), int(rp[r1])
                kw = dict(csr=(np.ascontiguousarray(rp[r0:r1 + 1] - lo), ci[lo:hi], va[lo:hi]))
            # each rank on its own stream (as one process per GPU would be)
            with T.TruncatedSVD(**kw, dist=dist, stream=torch.cuda.Stream()) as h:
                out[g] = _solve(h, algo)
        except Exception as ex:  # surfaced in the main thread
            err.append(ex)

    ths = [threading.Thread(target=rank_main, args=(g,)) for g in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=300)
    grp.close()
    assert not err, err
    assert all(o is not None for o in out)
    U = np.concatenate([o[1] for o in out])
    V = np.concatenate([o[3] for o in out])
    return out, U, V


def _case(kind):
    if kind == "dense":
        A = dense_prescribed(300, 120, spectrum_eq16(120), SEEDS["C1"])
        return A, 300, 120, dict(A=A)
    m, n = 6000, 4000
    csr = powerlaw_csr(m, n, 60000, 2.5, seed=9)
    return csr, m, n, dict(csr=csr, shape=(m, n))


@pytest.mark.parametrize("algo", ["lanczos", "rsvd", "thick", "pip2"])
@pytest.mark.parametrize("kind", ["dense", "csr"])
@pytest.mark.parametrize("world", [2, 3])
def test_loopback_world_equals_single(world, kind, algo):
    data, m, n, kw = _case(kind)
    with T.TruncatedSVD(**kw) as h:
        st1, U1, S1, V1, e1, info1, conv1 = _solve(h, algo)
    if kind == "csr":
        bounds = T.partition_rows(data[0], world)
    else:
        bounds = np.linspace(0, m, world + 1).astype(np.int64)
    out, U2, V2 = _run_world(kind, data, m, n, bounds, algo)
    c = conv1
    if algo == "rsvd":   # finite q: the iterate itself is the result (q = 2)
        c = np.ones_like(conv1)
    assert c.sum() >= 4
    for st2, _, S2, _, e2, info2, _ in out:
        assert st2 == st1
        assert info2["cycles"] == info1["cycles"]
        assert np.abs(S2 - S1)[c].max() <= 1e-12 * S1[0]
        assert np.abs(e2 - out[0][4]).max() == 0.0      # all-reduced: identical on all ranks
        assert np.abs(e2 - e1)[c].max() <= 1e-10
    assert U2.shape == U1.shape and V2.shape == V1.shape
    tolv = 1e-9 if algo != "rsvd" else 1e-7
    assert np.abs(U2 - U1)[:, c].max() <= tolv and np.abs(V2 - V1)[:, c].max() <= tolv
    # and against the oracle: the converged sigma of the single solve
    op = oracle.Operator(dense=data) if kind == "dense" else oracle.Operator(csr=data, shape=(m, n))
    eo, _ = oracle.residuals(op, U2, out[0][2], V2)
    assert np.abs(eo - out[0][4]).max() <= 1e-12


def test_loopback_empty_shard():
    """world 4 on a 9-column dense matrix split so that rank 3 has no rows
    and (ceil(9/4) = 3: shards 3, 3, 3, 0) no n-shard either: its Gram and
    projection partials must be zeros, not stale data."""
    rng = np.random.default_rng(3)
    m, n = 40, 9
    A = rng.standard_normal((m, n))
    with T.TruncatedSVD(A=A) as h:
        h.set_seed(2)
        st1 = h.block_lanczos(r=3, b=3, tol=1e-12, maxit=4, d=9)
        U1, S1, V1 = h.get()
    bounds = np.array([0, 15, 30, 40, 40])
    grp = T.LoopbackGroup(4)
    out = [None] * 4
    err = []

    def rank_main(g):
        try:
            torch.cuda.set_device(0)
            dist = dict(rank=g, world=4, nccl_id=None, loopback=grp, m_global=m, n_global=n,
                        row_begin=int(bounds[g]), row_end=int(bounds[g + 1]))
            with T.TruncatedSVD(A=np.ascontiguousarray(A[bounds[g]:bounds[g + 1]]), dist=dist,
                                stream=torch.cuda.Stream()) as h:
                h.set_seed(2)
                st = h.block_lanczos(r=3, b=3, tol=1e-12, maxit=4, d=9)
                out[g] = (st, *h.get())
        except Exception as ex:
            err.append(ex)

    ths = [threading.Thread(target=rank_main, args=(g,)) for g in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=120)
    grp.close()
    assert not err, err
    assert out[3][1].shape == (0, 3) and out[3][3].shape == (0, 3)
    U2 = np.concatenate([o[1] for o in out])
    V2 = np.concatenate([o[3] for o in out])
    assert out[0][0] == st1
    assert np.abs(out[0][2] - S1).max() <= 1e-12 * S1[0]
    assert np.abs(U2 - U1).max() <= 1e-9 and np.abs(V2 - V1).max() <= 1e-9

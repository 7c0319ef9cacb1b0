"""Multi-GPU decomposition on CPU: world_size 2 and 3 with the
gloo backend.  Each rank runs the row-partitioned LancSVD / RandSVD model
(oracle/dist.py: reduce-scatter of A^T Qbar, all-gather of Q_i, all-reduced
projections and Grams, Philox rows by global index, replicated small SVD)
on the row split chosen by the library's own host partitioner
(tsvd_partition_rows), and the gathered result must equal the single-process
oracle.  -m "not gpu"."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


_D = {"dense": 24, "csr": 96}  # Krylov dimension: both problems converge in a few cycles


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(kind):
    from tsvd_inputs import SEEDS, dense_prescribed, powerlaw_csr, spectrum_eq16
    if kind == "dense":
        s = spectrum_eq16(100)
        return dict(dense=dense_prescribed(200, 100, s, SEEDS["C1"]), m=200, n=100)
    csr = powerlaw_csr(3000, 2000, 30000, 2.5, seed=77)
    return dict(csr=csr, m=3000, n=2000)


def _worker(rank, world, port, kind, algo, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2403_06218_b200 as T
    from oracle import dist as od
    pb = _problem(kind)
    m, n = pb["m"], pb["n"]
    if "csr" in pb:
        bounds = T.partition_rows(pb["csr"][0], world)
    else:
        bounds = np.linspace(0, m, world + 1).astype(np.int64)
    comm = od.Comm()
    shard = od.RowShard(comm, m, n, bounds, csr=pb.get("csr"), dense=pb.get("dense"))
    if algo == "lanczos":
        U, S, V, cyc = od.lancsvd_dist(shard, r=8, b=4, d=_D[kind], tol=1e-10, maxit=6, seed=11)
    else:
        U, S, V = od.randsvd_dist(shard, r=8, p=8, q=2, b_qr=8, seed=11)
    Uf = comm.allgather_rows(U)
    Vf = comm.allgather_rows(V)
    if rank == 0:
        out.put((Uf, S, Vf, [int(x) for x in bounds]))
    dist.destroy_process_group()


def _run(world, kind, algo):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, kind, algo, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,kind,algo", [(2, "dense", "lanczos"), (2, "csr", "lanczos"),
                                             (3, "csr", "lanczos"), (2, "csr", "rsvd")])
def test_row_partitioned_matches_single(world, kind, algo):
    import oracle
    Uf, S, Vf, bounds = _run(world, kind, algo)
    pb = _problem(kind)
    op = oracle.Operator(dense=pb["dense"]) if "dense" in pb else \
        oracle.Operator(csr=pb["csr"], shape=(pb["m"], pb["n"]))
    if algo == "lanczos":
        ro = oracle.lancsvd(op, r=8, b=4, d=_D[kind], tol=1e-10, maxit=6, seed=11)
        assert ro.converged
    else:
        ro = oracle.randsvd(op, r=8, p=8, q=2, b_qr=8, seed=11)
    assert len(bounds) == world + 1 and bounds[0] == 0 and bounds[-1] == pb["m"]
    assert np.abs(S - ro.S).max() / ro.S[0] <= 1e-12
    gaps = np.minimum(np.abs(np.diff(np.r_[np.inf, ro.S])), np.abs(np.diff(np.r_[ro.S, -np.inf])))
    for i in range(8):
        if gaps[i] > 1e-3 * ro.S[0]:
            assert np.abs(Vf[:, i] - ro.V[:, i]).max() <= 1e-9
            assert np.abs(Uf[:, i] - ro.U[:, i]).max() <= 1e-9
    e, _ = oracle.residuals(op, Uf, S, Vf)
    assert np.abs(e - oracle.residuals(op, ro.U, ro.S, ro.V)[0]).max() <= 1e-9


def test_partition_rows_balanced():
    import paper_2403_06218_b200 as T
    from tsvd_inputs import powerlaw_csr
    rp, _, _ = powerlaw_csr(20000, 20000, 200000, 2.5, seed=3)
    for world in (1, 2, 4, 8):
        b = T.partition_rows(rp, world)
        assert b[0] == 0 and b[-1] == 20000 and np.all(np.diff(b) >= 0)
        nnz = np.diff(rp[b])
        assert nnz.max() - nnz.min() <= np.diff(rp).max() + 1

"""Host-side check of the split-grid algorithm on CPU.

Two processes (world_size 2, torch.distributed `gloo` on 127.0.0.1) run the
decomposition the CUDA path implements — the slab plan from the C-ABI
(`mprkb_slab_plan`), ghost-plane exchange with the send/receive order of
NcclComm::halo, the k-slab <-> j-slab transposes of FastDiagOp::apply_split
(peer-blocked rows, all-to-all), rank-ordered dot sums and the PARITY dot
chain — in numpy, and compare the gathered results with the single-domain
C oracle (oracle/mprk_oracle.c):
  * 7-point stencils (Dirichlet heat, periodic advection ring): bitwise;
  * the FastDiag stage preconditioner: 1e-12 relative (reordered sums);
  * the chained sequential fp32 dot: bitwise the global sequential sum.
No GPU is involved; the CUDA kernels are checked against the same oracle
on the B200 (tests/test_gpu_split.py).
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _halo(dist, rank, world, slab, periodic):
    """Exchange boundary planes like Comm::halo: my first plane -> lower's hi
    ghost, my last plane -> upper's lo ghost.  Tags keep a 2-rank ring
    (lower == upper) unambiguous."""
    lo = rank - 1 if rank > 0 else (world - 1 if periodic else -1)
    hi = rank + 1 if rank < world - 1 else (0 if periodic else -1)
    import torch

    glo = torch.zeros(slab.shape[1:], dtype=torch.from_numpy(slab).dtype)
    ghi = torch.zeros_like(glo)
    reqs = []
    if hi >= 0:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(slab[-1])), hi, tag=1))
    if lo >= 0:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(slab[0])), lo, tag=2))
    if lo >= 0:
        reqs.append(dist.irecv(glo, lo, tag=1))
    if hi >= 0:
        reqs.append(dist.irecv(ghi, hi, tag=2))
    for r in reqs:
        r.wait()
    return (glo.numpy() if lo >= 0 else None), (ghi.numpy() if hi >= 0 else None)


def _stencil_slab(x, glo, ghi, periodic, sigma, gamma):
    """The reference's per-point arithmetic (operators.hpp:133-158) on a slab
    padded with its ghost planes (zero = Dirichlet ghost)."""
    nz, n, _ = x.shape
    z = np.zeros((1, n, n), x.dtype)
    pad = np.concatenate([glo[None] if glo is not None else z, x, ghi[None] if ghi is not None else z])
    zm, zp = pad[:-2], pad[2:]
    if periodic:
        xl, xr = np.roll(x, 1, axis=2), np.roll(x, -1, axis=2)
        ym, yp = np.roll(x, 1, axis=1), np.roll(x, -1, axis=1)
        acc = xr - xl
        acc = acc + (yp - ym)
        acc = acc + (zp - zm)
    else:
        xl = np.concatenate([np.zeros((nz, n, 1), x.dtype), x[:, :, :-1]], axis=2)
        xr = np.concatenate([x[:, :, 1:], np.zeros((nz, n, 1), x.dtype)], axis=2)
        ym = np.concatenate([np.zeros((nz, 1, n), x.dtype), x[:, :-1, :]], axis=1)
        yp = np.concatenate([x[:, 1:, :], np.zeros((nz, 1, n), x.dtype)], axis=1)
        acc = x * 6.0
        for nb in (xl, xr, ym, yp, zm, zp):
            acc = acc - nb
    return sigma * x + gamma * acc


def _alltoall(dist, blocks):
    """all-to-all by all_gather (gloo): rank r keeps block r of every peer."""
    import torch

    world = dist.get_world_size()
    t = torch.from_numpy(np.ascontiguousarray(blocks))
    got = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(got, t)
    r = dist.get_rank()
    return np.stack([g.numpy()[r] for g in got])


def _worker(rank, world, port, n, out_q):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, ROOT)
    import paper_2412_16638_b200 as mp
    from oracle.oracle import Restatement

    O = Restatement()
    res = {}
    plan = mp.slab_plan(n, world, rank)
    k0, nz, j0, ny = plan["k0"], plan["nz"], plan["j0"], plan["ny"]
    rng = np.random.default_rng(4242)

    # ---- Dirichlet heat stencil (fp64) and periodic central stencil (c128)
    x = rng.uniform(-1, 1, n ** 3)
    slab = x.reshape(n, n, n)[k0:k0 + nz]
    glo, ghi = _halo(dist, rank, world, slab, periodic=False)
    mine = _stencil_slab(slab, glo, ghi, False, 1.0, -0.37)
    res["heat"] = (k0, mine.ravel(), O.stencil(1, n, 0, 1.0, -0.37, x))
    xc = rng.uniform(-1, 1, n ** 3) + 1j * rng.uniform(-1, 1, n ** 3)
    slab = xc.reshape(n, n, n)[k0:k0 + nz]
    glo, ghi = _halo(dist, rank, world, slab, periodic=True)
    mine = _stencil_slab(slab, glo, ghi, True, 1.0, 0.25)
    res["advection"] = (k0, mine.ravel(), O.stencil(3, n, 1, 1.0, 0.25, xc))

    # ---- FastDiag stage preconditioner (heat, fp64): FAST order of apply_split
    tau, a = 0.01, 0.5
    h = 1.0 / (n - 1)
    g = -tau * a * (-1.0 / h ** 2)
    qa, qai, la = O.spectral(0, n, 1.0, g)
    qb, qbi, lb = O.spectral(0, n, 0.0, g)
    qa, qai, qb, qbi = (m.reshape(n, n) for m in (qa, qai, qb, qbi))
    X = x.reshape(n, n, n)[k0:k0 + nz]                    # [kl][j][i]
    T = np.einsum("ai,kji->kja", qai, X)                  # R: Qa^-1
    T = np.einsum("bj,kji->kbi", qbi, T)                  # M: Qb^-1
    send = np.stack([T[:, s * ny:(s + 1) * ny, :] for s in range(world)])  # [s][kl][jl][i]
    J = _alltoall(dist, send).reshape(n, ny, n)           # [k][jl][i]
    pd = 1.0 / (la[None, None, :] + lb[j0:j0 + ny][None, :, None] + lb[:, None, None])
    J = np.einsum("ck,kji->cji", qbi, J) * pd             # L: Qc^-1 (Qc = Qb), * pd_inv
    J = np.einsum("ck,kji->cji", qb, J)                   # L: Qc
    back = _alltoall(dist, J.reshape(world, nz, ny, n))   # [r][kl][jl][i]
    K = np.concatenate(list(back), axis=1)                # [kl][j][i]
    K = np.einsum("bj,kji->kbi", qb, K)                   # M: Qb
    K = np.einsum("ai,kji->kja", qa, K)                   # R: Qa
    res["fastdiag"] = (k0, K.ravel(), O.fastdiag(1, n, tau, a, x))

    # ---- dots: FAST rank-ordered fp64 partials; PARITY chained fp32 accumulator
    import torch

    u = rng.uniform(-1, 1, n ** 3).astype(np.float32)
    v = rng.uniform(-1, 1, n ** 3).astype(np.float32)
    us, vs = u[k0 * n * n:(k0 + nz) * n * n], v[k0 * n * n:(k0 + nz) * n * n]
    part = torch.tensor([float(np.dot(us.astype(np.float64), vs.astype(np.float64)))], dtype=torch.float64)
    allp = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allp, part)
    fast = 0.0
    for p in allp:
        fast += float(p[0])
    acc = np.float32(0.0)
    for r in range(world):
        if r == rank:
            for a_, b_ in zip(us, vs):
                acc = np.float32(acc + np.float32(a_ * b_))
        t = torch.tensor([float(acc)], dtype=torch.float64)
        dist.broadcast(t, r)
        acc = np.float32(t.item())
    seq = np.float32(0.0)
    for a_, b_ in zip(u, v):
        seq = np.float32(seq + np.float32(a_ * b_))
    res["dot"] = (fast, float(np.dot(u.astype(np.float64), v.astype(np.float64))), float(acc), float(seq))
    out_q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 8), (2, 12)])
def test_split_algorithm_gloo(world, n):
    import multiprocessing as pmp

    pytest.importorskip("torch")
    ctx = pmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for key in ("heat", "advection", "fastdiag"):
        parts = sorted(results[r][key][:2] for r in range(world))
        got = np.concatenate([p[1] for p in sorted(parts, key=lambda t: t[0])])
        want = results[0][key][2]
        if key == "fastdiag":
            assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want), key
        elif key == "heat":
            assert np.array_equal(got, want), key
        else:
            assert np.allclose(got, want, rtol=0, atol=1e-15), key
    for r in range(world):
        fast, exact, chained, seq = results[r]["dot"]
        assert abs(fast - exact) <= 1e-13 * abs(exact)
        assert chained == seq  # the PARITY chain is the global sequential sum, bit for bit

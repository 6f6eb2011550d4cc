"""The NCCL split path with real processes: 2 ranks, one process each.

`gpurun` boxes have one GPU, and NCCL normally refuses two ranks on the same
device; when the local NCCL accepts it (or a second GPU is visible) this runs
the production transport — ncclSend/Recv halos, grouped all-to-all
transposes, all-gather scalar reductions — end to end and checks the split
PARITY step bitwise against the undivided one.  Otherwise it skips with
NCCL's reason (the same code paths run in-process in test_gpu_split.py and
through a 1-rank NCCL communicator in test_nccl_single_rank).
"""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rank(rank, world, uid_q, out_q):
    sys.path.insert(0, ROOT)
    import torch

    dev = rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    import paper_2412_16638_b200 as mp

    try:
        mp.set_device(dev)
        if rank == 0:
            uid = mp.Comm.nccl_unique_id()
            for _ in range(world - 1):
                uid_q.put(uid)
        else:
            uid = uid_q.get(timeout=60)
        comm = mp.Comm.nccl(rank, world, uid)
        res = {}
        for eq, method, prec, tol in (("heat", "4s3pB", "f32", 1e-4), ("advection", "4s3pC", "f64", 1e-8)):
            tab = mp.builtin(method)
            tau = 0.01 if eq == "heat" else 1.0 / 640.0
            st = mp.Stepper(eq, 16, tab, tau, tol, prec, 40, numerics="parity", comm=comm)
            u = st.initial_state()
            its = [st.step(u)["iterations"] for _ in range(2)]
            res[eq] = (st.k0, u, its)
            del st
        out_q.put((rank, "ok", res))
    except Exception as e:  # noqa: BLE001 - reported to the parent
        out_q.put((rank, "error", repr(e)))


def test_nccl_two_processes(gpu, mp):
    import multiprocessing as pmp

    ctx = pmp.get_context("spawn")
    uid_q, out_q = ctx.Queue(), ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, 2, uid_q, out_q)) for r in range(2)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(2):
            rank, status, payload = out_q.get(timeout=300)
            results[rank] = (status, payload)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    errors = [payload for status, payload in results.values() if status == "error"]
    if errors:
        if any("Duplicate GPU" in e or "invalid usage" in e.lower() for e in errors):
            pytest.skip(f"NCCL refuses two ranks on one GPU here: {errors[0][:200]}")
        raise AssertionError(errors)
    for eq, method, prec, tol in (("heat", "4s3pB", "f32", 1e-4), ("advection", "4s3pC", "f64", 1e-8)):
        tab = mp.builtin(method)
        tau = 0.01 if eq == "heat" else 1.0 / 640.0
        whole = mp.Stepper(eq, 16, tab, tau, tol, prec, 40, numerics="parity")
        w = whole.initial_state()
        wits = [whole.step(w)["iterations"] for _ in range(2)]
        parts = sorted((results[r][1][eq] for r in range(2)), key=lambda t: t[0])
        got = np.concatenate([p[1] for p in parts])
        assert all(p[2] == wits for p in parts)
        assert np.array_equal(got.view(np.uint64), w.view(np.uint64)), eq

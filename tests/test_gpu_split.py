"""Split grid (k-slab decomposition) on one B200.

The in-process communicator runs P ranks as threads sharing the GPU, so
every multi-rank code path — ghost-plane exchange before each stencil, the
FastDiag all-to-all transposes, rank-ordered Krylov reductions, collective
error flags — runs here exactly as it does across GPUs; only the transport
differs (device copies instead of NCCL over NVLink).

PARITY: the split run is BITWISE the undivided run (which the solver tests
pin bitwise to the reference): same stencil arithmetic per point, the
reference's contraction order around the transposes, and the sequential dot
accumulator carried from rank to rank in global index order.
FAST: within the tolerances the undivided FAST path itself meets
(fp64 1e-12 relative per step, fp32 within the fp32 stage noise), iteration
counts +-1.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run_split(mp, P, steps, make, backend="local"):
    """Step a split stepper on P in-process ranks; returns the global state
    (ranks' slabs concatenated), the per-step traces and rank 0's histories."""

    def body(rank, comm):
        st = make(comm)
        u = st.initial_state()
        traces, hists = [], []
        for _ in range(steps):
            tr = st.step(u)
            traces.append(tr)
            hists.append([st.history(i) for i in range(len(tr["iterations"]))])
        return st.k0, u, traces, hists

    res = mp.run_ranks(P, body)
    res.sort(key=lambda r: r[0])
    state = np.concatenate([r[1] for r in res])
    # every rank must report the same solver behaviour
    for r in res[1:]:
        assert [t["iterations"] for t in r[2]] == [t["iterations"] for t in res[0][2]]
    return state, res[0][2], res[0][3]


def run_whole(mp, steps, make):
    st = make(None)
    u = st.initial_state()
    traces, hists = [], []
    for _ in range(steps):
        tr = st.step(u)
        traces.append(tr)
        hists.append([st.history(i) for i in range(len(tr["iterations"]))])
    return u, traces, hists


def maker(mp, eq, n, method, prec, numerics, tol, max_iter=40, **kw):
    tab = mp.midpoint_corrected(1) if method == "midpoint1" else mp.builtin(method)
    tau = 0.01 if eq == "heat" else 1.0 / 640.0

    def make(comm):
        return mp.Stepper(eq, n, tab, tau, tol, prec, max_iter, numerics=numerics, comm=comm, **kw)

    return make


PARITY_CASES = [
    # eq, n, method, precision, tol, P
    ("heat", 16, "midpoint1", "f32", 1e-5, 2),
    ("heat", 16, "4s3pB", "f64", 1e-9, 4),
    ("heat", 16, "4s3pC", "f32", 1e-4, 1),
    ("heat", 12, "4s3pB", "f32", 1e-6, 3),   # multi-iteration fp32 CG, odd rank count
    ("advection", 16, "4s3pC", "f64", 1e-8, 2),
    ("advection", 16, "4s3pB", "f32", 1e-4, 4),
    ("advection", 12, "midpoint1", "f64", 1e-10, 1),
]


@pytest.mark.parametrize("eq,n,method,prec,tol,P", PARITY_CASES)
def test_split_parity_bitwise(gpu, mp, eq, n, method, prec, tol, P):
    make = maker(mp, eq, n, method, prec, "parity", tol)
    want, wtr, whist = run_whole(mp, 2, make)
    got, gtr, ghist = run_split(mp, P, 2, make)
    assert [t["iterations"] for t in gtr] == [t["iterations"] for t in wtr]
    assert [t["true_residual"] for t in gtr] == [t["true_residual"] for t in wtr]
    for hs, hw in zip(ghist, whist):
        for a, b in zip(hs, hw):
            assert np.array_equal(a, b)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (
        f"max |diff| {np.max(np.abs(got - want)):.3e}")


# fp32 tolerances: 2x the reference's own fp32 noise per step at 32^3
# (3.4e-6 for 4s3pB, 9.5e-5 for midpoint1, whose explicit
# corrector amplifies stage rounding by ~(tau |K|)^2 / 2)
FAST_CASES = [
    ("heat", 32, "4s3pB", "f64", 1e-9, 2, 1e-12),
    ("heat", 32, "4s3pB", "f32", 1e-4, 4, 2e-5),
    ("heat", 32, "midpoint1", "f32", 1e-5, 2, 1.9e-4),
    ("advection", 32, "4s3pC", "f64", 1e-8, 4, 1e-12),
    ("advection", 32, "4s3pC", "f32", 1e-3, 2, 2e-5),
]


@pytest.mark.parametrize("eq,n,method,prec,tol,P,rtol", FAST_CASES)
def test_split_fast_matches_undivided(gpu, mp, eq, n, method, prec, tol, P, rtol):
    make = maker(mp, eq, n, method, prec, "fast", tol)
    steps = 1 if method == "midpoint1" else 3
    want, wtr, _ = run_whole(mp, steps, make)
    got, gtr, _ = run_split(mp, P, steps, make)
    for a, b in zip(gtr, wtr):
        assert all(abs(x - y) <= 1 for x, y in zip(a["iterations"], b["iterations"]))
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel <= rtol, rel


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_split_fast_tensor_cores_256(gpu, mp, ranks):
    """The bench path on a split grid: fp32 FastDiag on tcgen05 in both slab
    layouts (k-slab R/M, j-slab L), 256^3 on 2 ranks.  Bar (SURVEY.md §8c,
    as test_step_fast_256_within_reference_noise): one step within 2x the
    fp32 policy's own distance from the fp64-policy step (which matches the
    reference to 1e-12)."""
    make = maker(mp, "heat", 256, "4s3pB", "f32", "fast", 1e-3)
    want, wtr, _ = run_whole(mp, 1, make)
    exact, _, _ = run_whole(mp, 1, maker(mp, "heat", 256, "4s3pB", "f64", "fast", 1e-5))
    got, gtr, _ = run_split(mp, ranks, 1, make)  # (M contractions on the peer-blocked layout: ny = 128 / 64)
    assert [t["iterations"] for t in gtr] == [t["iterations"] for t in wtr]
    own = np.linalg.norm(want - exact)
    assert np.linalg.norm(got - want) <= 2 * own, (np.linalg.norm(got - want), own)
    assert np.linalg.norm(got - exact) <= 2 * own


@pytest.mark.parametrize("ranks", [2, 4])
def test_split_config3_512(gpu, mp, ranks):
    """Config 3's size (BASELINE.json configs[2]: heat 512^3, k-slabs): one
    4s3pB fp32 FAST step on 2 / 4 in-process ranks against the undivided
    512^3 step, with the 256^3 test's bar — within 2x the fp32 policy's own
    distance from the fp64-policy step; iteration counts equal.  (The
    reference needs ~18 min per 4s3pB step at 512^3 on 8 cores, SURVEY.md
    §8d, so the size-independent split-vs-undivided property is the check.)"""
    make = maker(mp, "heat", 512, "4s3pB", "f32", "fast", 1e-3)
    want, wtr, _ = run_whole(mp, 1, make)
    exact, _, _ = run_whole(mp, 1, maker(mp, "heat", 512, "4s3pB", "f64", "fast", 1e-5))
    got, gtr, _ = run_split(mp, ranks, 1, make)
    assert [t["iterations"] for t in gtr] == [t["iterations"] for t in wtr]
    own = np.linalg.norm(want - exact)
    assert own > 0
    assert np.linalg.norm(got - want) <= 2 * own, (np.linalg.norm(got - want), own)
    assert np.linalg.norm(got - exact) <= 2 * own


def test_split_block_jacobi_fp16(gpu, mp):
    """Multi-iteration CG with the block-Jacobi extension (x-line blocks stay
    inside a slab) and fp16 block storage."""
    make = maker(mp, "heat", 32, "4s3pB", "f32", "fast", 1e-5, preconditioner="block-jacobi", block_size=8,
                 block_storage="f16", max_iter=300)
    want, wtr, _ = run_whole(mp, 1, make)
    got, gtr, _ = run_split(mp, 4, 1, make)
    assert all(abs(x - y) <= 1 for x, y in zip(gtr[0]["iterations"], wtr[0]["iterations"]))
    assert min(wtr[0]["iterations"]) > 5
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel <= 1e-4, rel


def test_split_integrate_errors(gpu, mp):
    """integrate() on a split grid: the global error norms (max / RMS over all
    ranks) match the undivided run."""
    tab = mp.builtin("4s3pB")
    n = 16
    whole = mp.Stepper("heat", n, tab, 0.01, 1e-9, "f64", 40, t_end=0.05).integrate()

    def body(rank, comm):
        st = mp.Stepper("heat", n, tab, 0.01, 1e-9, "f64", 40, t_end=0.05, comm=comm)
        r = st.integrate()
        return r["error_max"], r["error_l2"], r["solve_iterations"]

    res = mp.run_ranks(2, body)
    for em, el, its in res:
        assert its == whole["solve_iterations"]
        assert abs(em - whole["error_max"]) <= 1e-12 * whole["error_max"]
        assert abs(el - whole["error_l2"]) <= 1e-12 * whole["error_l2"]


def test_split_errors_raised_on_every_rank(gpu, mp):
    """A non-finite state on one rank's slab raises NonFiniteState on all
    ranks (collective flags), not a hang."""
    tab = mp.builtin("4s3pB")

    def body(rank, comm):
        st = mp.Stepper("heat", 16, tab, 0.01, 1e-6, "f64", 40, comm=comm)
        u = st.initial_state()
        if rank == 1:
            u[5] = np.nan
        try:
            st.step(u)
        except mp.NonFiniteState:
            return "raised"
        return "no error"

    assert mp.run_ranks(2, body) == ["raised", "raised"]


@pytest.mark.parametrize("gate", ["device", "host"])
def test_split_fused_step_error_leaves_every_slab_untouched(gpu, mp, gate):
    """The fused fp32 split step gates its final update on the OR of every
    rank's stage checks (all-gathered on the stream; MPRKB_SPLIT_GATE=0: the
    host decides before the update): a NaN in one rank's slab raises
    NonFiniteState on every rank and no rank's state is modified."""
    import os

    tab = mp.builtin("4s3pB")

    def body(rank, comm):
        st = mp.Stepper("heat", 256, tab, 0.01, 1e-3, "f32", 40, comm=comm)
        u = st.initial_state() + 0.5
        if rank == 1:
            u[12345] = np.nan
        u0 = u.copy()
        try:
            st.step(u)
        except mp.NonFiniteState:
            return "raised", np.array_equal(u, u0, equal_nan=True)
        return "no error", False

    if gate == "host":
        os.environ["MPRKB_SPLIT_GATE"] = "0"
    try:
        res = mp.run_ranks(2, body)
    finally:
        os.environ.pop("MPRKB_SPLIT_GATE", None)
    assert res == [("raised", True), ("raised", True)]


def test_split_rejects_uneven_slabs(gpu, mp):
    tab = mp.builtin("4s3pB")

    def body(rank, comm):
        with pytest.raises(ValueError):
            mp.Stepper("heat", 10, tab, 0.01, 1e-6, "f64", 40, comm=comm)
        return True

    assert all(mp.run_ranks(3, body))


def test_nccl_single_rank(gpu, mp):
    """The NCCL backend (one process per GPU) on the one GPU a box has: a
    1-rank communicator still routes every exchange through the split path
    (self all-to-all, self ring halo, NCCL all-gather of the Krylov scalars)."""
    uid = mp.Comm.nccl_unique_id()
    comm = mp.Comm.nccl(0, 1, uid)
    assert np.array_equal(comm.allreduce_sum([1.5, -2.0]), [1.5, -2.0])
    for eq, method, prec, tol, numerics in (("heat", "4s3pB", "f32", 1e-4, "parity"),
                                            ("advection", "4s3pC", "f64", 1e-8, "fast")):
        make = maker(mp, eq, 16, method, prec, numerics, tol)
        want, wtr, _ = run_whole(mp, 2, make)
        st = make(comm)
        u = st.initial_state()
        for _ in range(2):
            tr = st.step(u)
        assert tr["iterations"] == wtr[-1]["iterations"]
        if numerics == "parity":
            assert np.array_equal(u, want)
        else:
            assert np.linalg.norm(u - want) <= 1e-12 * np.linalg.norm(want)
        del st



@pytest.mark.parametrize("ranks,tol", [(2, 1e-3), (4, 1e-3), (2, 1e-7)])
def test_split_speculative_stage_solves_bitwise(gpu, mp, ranks, tol):
    """Split grids speculate like the undivided grid: each solve's judge adds
    the ranks' all-gathered local sums (||r0||^2, p.Ap, r.z, ||r1||^2,
    ||b - A x1||^2) in rank order on the device, so the step needs no round
    trip per solve; states, iteration counts and residual histories are
    bitwise the round-trip path (MPRKB_SPLIT_SPECULATE=0).  tol 1e-7 forces
    misses (the one-iteration exit fails, the step is redone with round trips)."""
    import os

    make = maker(mp, "heat", 256, "4s3pB", "f32", "fast", tol)
    a, ta, ha = run_split(mp, ranks, 2, make)
    os.environ["MPRKB_SPLIT_SPECULATE"] = "0"
    try:
        b, tb, hb = run_split(mp, ranks, 2, make)
    finally:
        os.environ.pop("MPRKB_SPLIT_SPECULATE", None)
    assert [t["iterations"] for t in ta] == [t["iterations"] for t in tb]
    if tol > 1e-5:
        assert all(i == 1 for t in ta for i in t["iterations"])
    else:
        assert max(i for t in ta for i in t["iterations"]) > 1
    for x, y in zip(ha, hb):
        for hx, hy in zip(x, y):
            assert np.array_equal(np.asarray(hx), np.asarray(hy))
    assert np.array_equal(a, b)


@pytest.mark.parametrize("ranks", [2, 4])
def test_split_device_alpha_bitwise_host_alpha(gpu, mp, ranks):
    """On a split grid the fused first CG update takes alpha from the ranks'
    all-gathered local (p.Ap, r.z) pairs, completed in rank order on the
    device (Comm::allgather_dev, one round trip per solve); bitwise the path
    that waits for the host's allreduced scalars (MPRKB_SPLIT_DEVALPHA=0)."""
    import os

    make = maker(mp, "heat", 256, "4s3pB", "f32", "fast", 1e-3)
    a, ta, _ = run_split(mp, ranks, 2, make)
    os.environ["MPRKB_SPLIT_DEVALPHA"] = "0"
    try:
        b, tb, _ = run_split(mp, ranks, 2, make)
    finally:
        os.environ.pop("MPRKB_SPLIT_DEVALPHA", None)
    assert [t["iterations"] for t in ta] == [t["iterations"] for t in tb]
    assert np.array_equal(a, b)

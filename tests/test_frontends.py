"""§8(f) front-ends around the path: the reference's CLI harness
(tools/main.cpp -> tools/mprk-b200), temporal_order (stepper.cpp:271-310)
and tableau JSON I/O (tableau.cpp:192-233).

CPU tests: the CLI builds, refuses without a device (no CPU fallback) and
validates its options; tableau JSON round-trips with the reference's error
messages.  GPU tests: run / convergence / bench / verify output formats and
values; temporal_order in PARITY numerics is bitwise the reference's.
"""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "mprk-b200")

RUN_KEYS = ["method", "equation", "n", "tau", "tend", "tol", "implicit_precision", "failed", "final_error_max",
            "final_error_l2", "mean_iterations", "total_iterations", "steps", "wall_seconds", "timings"]


def cli(*args):
    if not os.path.exists(CLI):
        subprocess.run(["make", "-C", ROOT, "tools/mprk-b200"], check=True, capture_output=True)
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


def test_cli_usage_and_no_fallback():
    r = cli()
    assert r.returncode == 1 and "subcommand" in r.stderr
    r = cli("run")
    assert r.returncode == 1 and "--method" in r.stderr
    r = cli("run", "--method", "4s3pB", "--prec", "f16")
    assert r.returncode == 1
    r = cli("stability", "--method", "4s3pB")
    assert r.returncode == 1 and "outside the B200 hot path" in r.stderr
    import torch

    if not torch.cuda.is_available():
        r = cli("run", "--method", "4s3pB")
        assert r.returncode == 1 and "no CUDA device" in r.stderr


def test_tableau_json_roundtrip(mp):
    t = mp.Tableau("user", 2, [0.5, 1.0], [[0, 0], [0.5, 0]], [[0.5, 0], [0, 0.0]], [0.5, 0.5])
    back = mp.tableau_from_json(mp.tableau_to_json(t))
    assert (back.name, back.q, back.c, back.a_high, back.a_eps, back.b) == (t.name, t.q, t.c, t.a_high, t.a_eps,
                                                                        t.b)
    no_c = json.loads(mp.tableau_to_json(t))
    del no_c["c"]
    assert mp.tableau_from_json(json.dumps(no_c)).c == [0.5, 0.5]  # derived: row sums of A_high + A_eps
    with pytest.raises(mp.MprkError, match="does not parse"):
        mp.tableau_from_json("{")
    with pytest.raises(mp.MprkError, match="wrong field"):
        mp.tableau_from_json('{"name": "x"}')
    bad = json.loads(mp.tableau_to_json(t))
    bad["b"] = [1.0]
    with pytest.raises(mp.MprkError, match="inconsistent with q"):
        mp.tableau_from_json(json.dumps(bad))


@pytest.mark.gpu
def test_cli_run_record(gpu, mp):
    r = cli("run", "--method", "4s3pB", "--n", "16", "--tau", "0.025", "--tend", "0.1", "--tol", "1e-6",
            "--prec", "f32")
    assert r.returncode == 0, r.stderr
    rec = json.loads(r.stdout)
    assert list(rec) == RUN_KEYS
    want = mp.integrate(mp.builtin("4s3pB"), "heat", 16, 0.025, 0.1, 1e-6, "f32")
    assert rec["steps"] == 4 and rec["failed"] is False
    assert rec["final_error_max"] == want["error_max"]
    assert rec["total_iterations"] == want["total_iterations"]
    assert rec["timings"]["solver"]["count"] == 16  # 4 steps x 4 implicit stages
    assert set(rec["timings"]) >= {"solver", "precond", "stencil", "axpy"}
    # the unstable default refusal (main.cpp:113-121)
    r = cli("run", "--method", "4s3pA")
    assert r.returncode == 1 and "unstable" in r.stderr


@pytest.mark.gpu
def test_cli_convergence_and_bench(gpu, mp):
    r = cli("convergence", "--method", "midpoint1", "--n", "8", "--tau", "0.025", "--tend", "0.1")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().split("\n")
    assert lines[0] == "tau,error_max,error_l2,order_running" and len(lines) == 5
    assert lines[1].endswith(",nan")
    orders = [float(x.split(",")[3]) for x in lines[2:]]
    assert all(1.5 < o < 2.5 for o in orders), orders  # second-order method
    r = cli("bench", "--method", "4s3pB", "--n", "16", "--repeat", "2")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().split("\n")
    assert lines[0] == "label,count,total_seconds,seconds_per_call"
    assert lines[-1].startswith("iterations,")
    rows = {x.split(",")[0]: x.split(",") for x in lines[1:]}
    assert int(rows["solver"][1]) == 2 * 4 * 4
    assert cli("verify").returncode == 0
    assert cli("verify", "--corrupt").returncode == 3


@pytest.mark.gpu
def test_temporal_order_parity_bitwise(gpu, mp, ref):
    """temporal_order in PARITY numerics: every run is bitwise the reference's,
    so the errors and the fitted slope are too."""
    t = mp.midpoint_corrected(1)
    tab = dict(q=t.q, a_high=np.array(t.a_high), a_eps=np.array(t.a_eps), b=np.array(t.b))
    taus = [0.025, 0.0125, 0.00625]
    got = mp.temporal_order(t, "heat", 8, taus, t_end=0.1, tol=1e-8, precision="f64", numerics="parity")
    want = ref.temporal_order(0, 8, tab, taus, 0.1, 1e-8, "f64")
    assert got["errors_max"] == want["errors_max"]
    assert got["errors_l2"] == want["errors_l2"]
    assert got["slope"] == want["slope"]
    assert got["solver_failure"] == want["solver_failure"]
    fast = mp.temporal_order(t, "heat", 8, taus, t_end=0.1, tol=1e-8, precision="f64")
    assert abs(fast["slope"] - want["slope"]) <= 1e-6 * abs(want["slope"])

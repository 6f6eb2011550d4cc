"""The reference's OWN C++ test suites run against the B200 library.

/root/reference/proj/tests/{test_krylov,test_precond,test_operators,
test_stepper,test_tableau,test_linalg,acceptance}.cpp are compiled UNMODIFIED
(`make refsuites`) with the include path pointed at the drop-in headers
include/mprk/ (the reference's API and namespace, backed by libmprk_b200.so)
and tests/cpp/doctest/doctest.h in place of doctest.  Every assertion of those
files then exercises the B200 kernels: KronSumOperator::apply, apply_tensor,
FastDiagPreconditioner, cg/gmres through the ApplyFn slot, Stepper::step,
integrate, temporal_order, the precision-isolation counters and the timing
labels.  The binaries are built in the build container (the reference sources
are not on the GPU box) and travel with the snapshot.
"""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SUITES = os.path.join(HERE, "cpp", "_ref_suites")
DEVICE = ["test_krylov", "test_precond", "test_operators", "test_stepper"]
HOST = ["test_tableau", "test_linalg"]


def _run(name, timeout=900):
    exe = os.path.join(SUITES, name)
    if not os.path.exists(exe):
        pytest.fail(f"{exe} missing: run `make refsuites` where /root/reference exists")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=timeout)
    return r


@pytest.mark.gpu
@pytest.mark.parametrize("name", DEVICE + HOST)
def test_reference_suite_on_b200(name):
    r = _run(name)
    tail = "\n".join(r.stdout.strip().splitlines()[-40:])
    assert r.returncode == 0 and "Status: SUCCESS" in r.stdout, tail


# criterion 3 (binary16 truncation of 4s3pA's stability region) FAILS in the
# reference itself as built here: its own stability.cpp + tableau.cpp give
# 33424 stable cells untruncated and 33428 under binary16 (checked with the
# reference sources compiled by g++ 13.3 in the build container), so the gate
# cannot exit 0 for the reference either.  The drop-in must reproduce exactly
# that outcome; every other criterion must pass.
REFERENCE_CRITERION_3 = "stable cells untruncated 33424, f16 33428, f32 33424"


@pytest.mark.gpu
def test_reference_acceptance_gate_on_b200():
    r = _run("acceptance", timeout=1800)
    lines = {int(l.split()[1]): l for l in r.stdout.splitlines() if l.startswith("criterion")}
    assert sorted(lines) == list(range(1, 12)), r.stdout[-4000:]
    for crit, line in lines.items():
        if crit == 3:
            assert "[FAIL]" in line and REFERENCE_CRITERION_3 in line, line
        else:
            assert "[PASS]" in line, line
    # criteria 6-8 (acceptance.cpp:213-279) are the iteration-count contract
    # of the stage solves, 9-10 temporal orders and F32 accuracy, 11 the
    # tensor-l / tensor-m timing labels


@pytest.mark.parametrize("name", HOST)
def test_reference_host_suites(name):
    """Suites that need no device (tableaus, spectral factors) also run here."""
    if not os.path.exists(os.path.join(SUITES, name)):
        pytest.skip("reference suites not built (make refsuites)")
    r = _run(name)
    assert r.returncode == 0 and "Status: SUCCESS" in r.stdout, r.stdout[-3000:]

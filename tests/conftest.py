import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference, ensure_built, have_reference

    ensure_built(ref=True)
    if not have_reference():
        pytest.skip("oracle/_ref/libmprk_ref.so not built (reference sources absent)")
    return Reference()


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Restatement, ensure_built

    ensure_built(ref=False)
    return Restatement()


@pytest.fixture(scope="session")
def mp():
    import paper_2412_16638_b200 as mp

    return mp


@pytest.fixture(scope="session")
def dropin_exe(tmp_path_factory, mp):
    """tests/cpp/dropin_example.cpp built against include/mprk_b200.hpp and
    linked to libmprk_b200.so (the C++ drop-in boundary)."""
    import subprocess

    exe = tmp_path_factory.mktemp("dropin") / "dropin"
    libdir = os.path.join(ROOT, "paper_2412_16638_b200")
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp"), "-o", str(exe),
                        "-L", libdir, "-lmprk_b200", "-Wl,-rpath," + libdir], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


@pytest.fixture(scope="session")
def gpu(mp):
    # -m gpu runs on the B200 box: a missing device is a failure, not a skip
    assert mp.device_count() >= 1, "no CUDA device visible to libmprk_b200.so"
    import torch

    assert torch.cuda.is_available()
    return torch.device("cuda:0")

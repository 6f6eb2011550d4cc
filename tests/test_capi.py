"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/mprk_b200.h declares, reports errors with the reference's
exception hierarchy, and refuses to compute without a device (no CPU
fallback).  No compute calls are made here."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mprk_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mprkb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(mp):
    lib = ctypes.CDLL(mp._c.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the python binding declares a signature for each of them
    assert set(syms) <= set(mp._c.SIGNATURES)


def test_library_is_sm100a_only(mp):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", mp._c.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "mprk_b200.h"\nint main(void){mprkb_config c; mprkb_config_init(&c); return c.max_iter;}\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-c", "-I", os.path.join(ROOT, "include"),
                        str(src), "-o", str(tmp_path / "t.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_config_defaults_match_reference(mp):
    """IntegrationConfig defaults (stepper.hpp:26-33): t_end 0.1, tol 1e-6, max_iter 40, F64."""
    cfg = mp._c.Config()
    mp._c.lib.mprkb_config_init(ctypes.byref(cfg))
    assert (cfg.t_end, cfg.tol, cfg.max_iter, cfg.implicit_precision) == (0.1, 1e-6, 40, mp._c.F64)


def test_no_device_means_error_not_fallback(mp):
    if mp.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(mp.NoDevice):
        mp.Stepper("heat", 8, mp.builtin("4s3pB"), 0.025)
    with pytest.raises(mp.NoDevice):
        mp.integrate(mp.builtin("4s3pB"), "heat", 8, 0.025, 0.1)


def test_argument_errors_map_like_the_reference(mp):
    """bindings.cpp:19-35 (ValueError) and stepper.cpp:220-225 (MprkError), no device needed."""
    t = mp.builtin("4s3pB")
    with pytest.raises(ValueError):
        mp.integrate(t, "plasma", 8, 0.025, 0.1)
    with pytest.raises(ValueError):
        mp.integrate(t, "heat", 8, 0.025, 0.1, precision="f8")
    with pytest.raises(mp.MprkError):
        mp.integrate(t, "heat", 8, 0.03, 0.1)
    with pytest.raises(mp.MprkError):
        mp.integrate(t, "heat", 8, -0.01, 0.1)
    with pytest.raises(mp.DimensionTooSmall):
        mp.integrate(t, "heat", 1, 0.025, 0.1)
    with pytest.raises(mp.MprkError):
        mp.builtin("4s3pD")
    assert issubclass(mp.DimensionTooSmall, mp.MprkError)


def test_cpp_dropin_header_builds_and_links(dropin_exe):
    """include/mprk_b200.hpp (the C++ drop-in for mprk::Stepper / integrate)
    compiles against the C-ABI and links against libmprk_b200.so."""
    assert dropin_exe.exists()

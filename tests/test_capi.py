"""The drop-in boundary without a GPU: libldg_b200.so loads, exports every
symbol include/ldg_b200.h declares, its host-side reference-element math
matches the reference fixtures, and the device path fails loudly (no CPU
fallback) where no GPU exists."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ldg_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ldg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_1408_3877_b200 as ld

    path = ld.library_path()
    assert os.path.exists(path), "build() must produce paper_1408_3877_b200/libldg_b200.so"
    lib = ctypes.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding declares exactly the ABI of the header
    assert sorted(ld._SIGNATURES) == syms
    nm = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r" T (ldg_[a-z0-9_]+)$", nm, flags=re.M)))
    assert exported == syms


def test_library_is_sm100a():
    import paper_1408_3877_b200 as ld

    out = subprocess.run(["cuobjdump", "--list-elf", ld.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n", [1, 3, 6, 10, 15])
def test_host_reference_tensors_match_reference(n, golden):
    """The product's own host math (table-driven basis, Newton Gauss rules) against
    build_ref_tensors of the unmodified reference (tests/golden/tensors.npz)."""
    import paper_1408_3877_b200 as ld

    g = golden("tensors")
    t = ld.reference_tensors(n)
    for key in ("m", "h", "g", "sd", "so", "rd", "ro"):
        ref = g[f"N{n}_{key}"]
        err = np.abs(t[key] - ref).max()
        assert err <= 4e-14 * max(1.0, np.abs(ref).max()), (key, err)


def test_invalid_order_rejected_without_gpu():
    import paper_1408_3877_b200 as ld

    with pytest.raises(ValueError):
        ld.reference_tensors(4)


def _have_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_have_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    import paper_1408_3877_b200 as ld

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        ld.LdgSystem.square(4, 1, ld.BASELINE_SPEC)


SIM = os.path.join(ROOT, "tools", "ldg_simulate")


@pytest.mark.skipif(_have_gpu(), reason="checks the no-GPU failure mode")
def test_cpp_host_mirror_fails_loudly_without_gpu():
    """tools/ldg_simulate (C++ mirror of cmd_simulate over ldg_host.hpp) maps the
    C ABI status to the reference's exit behaviour (ldg_main.cpp:302-305)."""
    assert os.path.exists(SIM), "build() must produce tools/ldg_simulate"
    r = subprocess.run([SIM, "4", "1", "2"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1
    assert "no CPU fallback" in r.stderr


@pytest.mark.parametrize("n", [1, 3, 6, 10, 15])
def test_rank_form_guard(n):
    """The rank-Q_e operator kernels are used only for tensors with the structure they
    assume (ldg_rank_form_supported, host-only): the library's own tensors have it, the
    reference's (golden) tensors have it, tensors with a perturbed s_offdiag or a filled
    upper part of h_hat do not."""
    import paper_1408_3877_b200 as ld

    assert ld.rank_form_supported(n)
    t = ld.reference_tensors(n)
    assert ld.rank_form_supported(n, t)
    bad = {k: v.copy() for k, v in t.items()}
    bad["so"][0] += 1e-9
    assert not ld.rank_form_supported(n, bad)
    bad = {k: v.copy() for k, v in t.items()}
    bad["h"].reshape(n, n, 2)[0, n - 1, 0] += 1e-9  # deg(phi_0) = 0 <= deg(phi_{n-1})
    assert not ld.rank_form_supported(n, bad)

"""The drop-in boundary exercised from the reference's side: a C++ program written
against the reference's own API (tests/cpp/dropin_reference_api.cpp) builds the
reference ComposedSolver and, through the adapter of INTEGRATION.md over
include/f3r_gpu.hpp, the device one, and solves the same system with both."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_reference_api")


def _have():
    return os.path.exists(BIN)


def test_dropin_binary_links():
    """CPU: the binary exists (built from the reference headers here) and every
    shared library it needs resolves (libf3r_ref + libf3rg via $ORIGIN rpaths)."""
    if not _have():
        pytest.skip("oracle/_ref/dropin_reference_api not built (needs /root/reference at build time)")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "not found" not in out, out
    assert "libf3rg.so" in out and "libf3r_ref.so" in out


def _run(lg, beta, spec=None, m=None):
    args = [BIN, str(lg), str(beta)] + ([spec] if spec else []) + ([m] if m else [])
    r = subprocess.run(args, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, OMP_NUM_THREADS=str(os.cpu_count() or 1)))
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("lg,beta", [(5, 0.0), (5, 0.5)])
def test_dropin_same_answer_as_reference(lg, beta):
    if not _have():
        pytest.skip("dropin binary not built")
    d = _run(lg, beta)
    assert d["id_cpu"] == d["id_gpu"]
    assert d["cpu"]["converged"] == 1 and d["gpu"]["converged"] == 1, d
    assert d["gpu"]["res"] <= 1e-10, d
    oc, og = d["cpu"]["outer"], d["gpu"]["outer"]
    assert abs(og - oc) <= max(1, round(0.1 * oc)), d
    # both solutions meet 1e-10 relative residual on a unit-diagonal SPD-ish system
    assert d["x_rel_diff"] < 1e-7, d
    assert d["parse_error_is_f3r"] == 1, d


@pytest.mark.gpu
@pytest.mark.parametrize("lg,beta,m", [(5, 0.0, "ic0"), (5, 0.5, "ilu0")])
def test_dropin_with_block_jacobi_m(lg, beta, m):
    """the reference bench's default M (block-Jacobi IC(0)/ILU(0), 4 blocks, fp16)
    handed to the adapter, which refactorises it on the device"""
    if not _have():
        pytest.skip("dropin binary not built")
    spec = f"F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > {m}(blocks=4,prec=f16)"
    d = _run(lg, beta, spec, m)
    assert d["id_cpu"] == d["id_gpu"]
    assert d["cpu"]["converged"] == 1 and d["gpu"]["converged"] == 1, d
    assert d["gpu"]["res"] <= 1e-10, d
    oc, og = d["cpu"]["outer"], d["gpu"]["outer"]
    assert abs(og - oc) <= max(1, round(0.1 * oc)), d
    assert d["x_rel_diff"] < 1e-7, d

"""CPU: the C-ABI library loads and exports every function include/*.h declares;
host-only entry points (spec grammar, problem generation, error reporting) work
without a GPU. No compute call is made here."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(f3rg_[a-z0-9_]+)\s*\(", src)))


@pytest.mark.parametrize("header", ["f3rg.h", "f3rg_problems.h"])
def test_every_declared_symbol_is_exported(header):
    import paper_2505_20719_b200 as f
    L = f.lib()
    names = declared(header)
    assert len(names) >= 4
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_product_library_has_no_cpu_fallback_symbols():
    """the product .so must not link the oracle or the reference"""
    import paper_2505_20719_b200 as f
    L = f.lib()
    for sym in ("or_spmv", "or_solve", "ref_solve", "ref_spmv"):
        assert not hasattr(L, sym)


def test_version_and_errors_without_gpu():
    import paper_2505_20719_b200 as f
    L = f.lib()
    assert b"sm_100a" in L.f3rg_version()
    with pytest.raises(f.ParseError) as e:
        f.canonical_spec("F8:f32")
    assert "F8:f32" in str(e.value)


def test_default_run_options_match_reference():
    import paper_2505_20719_b200 as f

    class Opts(C.Structure):
        _fields_ = [("tol", C.c_double), ("max_outer_restarts", C.c_int32), ("max_outer_total", C.c_uint64),
                    ("reset", C.c_int32)]
    o = Opts()
    f.lib().f3rg_default_run_options(C.byref(o))
    # include/f3r/nesting.hpp:29-38
    assert (o.tol, o.max_outer_restarts, o.max_outer_total, o.reset) == (1e-8, 3, 300, 0)
    r = f.RunOptions()
    assert (r.tol, r.max_outer_restarts, r.max_outer_total, r.reset_richardson_on_restart) == (1e-8, 3, 300, False)


def test_f3r_spec_matches_reference_preset():
    """f3r_spec (src/nesting.cpp:359-386) canonical ids for the three modes"""
    import paper_2505_20719_b200 as f
    assert f.f3r_spec(f.F3rConfig()).to_string() == \
        "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > ilu0(prec=f16)"
    assert f.f3r_spec(f.F3rConfig(mode=f.F3rMode.FP32)).to_string() == \
        "F100:f64/f64 > F8:f32/f32 > F4:f32/f32 > R2:f32,c=64 > ilu0(prec=f32)"
    assert f.f3r_spec(f.F3rConfig(mode=f.F3rMode.FP64, m1=50)).to_string() == \
        "F50:f64/f64 > F8:f64/f64 > F4:f64/f64 > R2:f64,c=64 > ilu0(prec=f64)"

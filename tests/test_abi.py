"""Host-side checks of the C ABI (no GPU needed): the library builds and loads, exports every
function include/h2.h declares, and rejects invalid arguments before touching a device."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    import paper_2206_01885_b200 as P
    from paper_2206_01885_b200 import build
    build.build()
    return P


def declared_functions():
    src = open(os.path.join(ROOT, "include", "h2.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(h2_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for f in ("h2_build", "h2_matvec", "h2_free"):
        assert f in names


def test_library_exports_every_declared_symbol(P):
    L = P.lib()
    names = declared_functions()
    assert len(names) >= 10
    for f in names:
        assert hasattr(L, f), f
    assert sorted(P.EXPORTED_SYMBOLS) == names


def test_options_default(P):
    o = P.h2_options_default()
    assert o.r_override == 0 and o.storage == P.H2_STORE_AUTO and not o.stream and o.points_on_host == 0


@pytest.mark.parametrize("args,code", [
    (dict(n=0), -1), (dict(d=0), -1), (dict(d=9), -1), (dict(q=0), -1), (dict(tau=0.0), -1), (dict(tau=0.8), -1),
    (dict(tol=0.0), -1), (dict(tol=1.0), -1), (dict(kid=8), -3), (dict(kid=0), -3), (dict(kid=2, kp=(-1.0,)), -1),
    (dict(kid=3, kp=(0.0,)), -1), (dict(kid=7), -1), (dict(kid=7, kp=(-100.0,)), -1)])
def test_invalid_arguments_rejected(P, args, code):
    a = dict(n=100, d=3, kid=1, kp=(), tol=1e-6, q=16, tau=0.5)
    a.update(args)
    L = P.lib()
    kp = (C.c_double * 1)(*(a["kp"] or (0.0,)))
    dummy = (C.c_double * 8)()
    h = L.h2_build(C.cast(dummy, C.c_void_p), a["n"], a["d"], a["kid"], kp if a["kp"] else None, a["tol"], a["q"],
                   a["tau"])
    assert not h
    assert L.h2_last_error() == code
    assert len(L.h2_last_error_message()) > 0


def test_null_safe_calls(P):
    L = P.lib()
    L.h2_free(None)
    assert L.h2_matvec(None, None, None) == -1
    assert L.h2_info(None, None) == -1
    assert L.h2_export(None, 1, None, 0, None) == -1


@pytest.mark.parametrize("reduct,d", [(3, 3), (-1, 3), (2, 5), (2, 1)])
def test_invalid_reduct_rejected(P, reduct, d):
    """h2_options.reduct outside H2_REDUCT_*, or the surface reduction with d not in {2, 3}."""
    L = P.lib()
    o = P.h2_options_default()
    o.reduct = reduct
    dummy = (C.c_double * 8)()
    h = L.h2_build_ex(C.cast(dummy, C.c_void_p), 100, d, 1, None, 1e-6, 16, 0.5, C.byref(o))
    assert not h
    assert L.h2_last_error() == -1

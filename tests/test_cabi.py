"""C-ABI library: loads, exports every symbol declared in include/ctrecon.h,
host-only functions behave (no GPU compute here)."""
import os
import re

import pytest

from oracle import alg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ctrecon.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s+\**([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def C():
    import __graft_entry__ as ge
    ge.build()
    from paper_1512_04564_b200 import ctrecon
    ctrecon.load()
    return ctrecon


def test_header_symbols_exported(C):
    names = header_functions()
    assert len(names) >= 16, names
    L = C.load()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(C.EXPORTS) == names


def test_rho_host_function_matches_eq37(C):
    for k in (0, 1, 2, 3, 10, 100, 719):
        for a in (1.0, 1.5, 1.999):
            assert abs(C.oslalm_rho(k, a) - alg.rho_k(k, a)) <= 1e-15


def test_no_gpu_fails_loudly(C):
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from synth.configs import get_config
    with pytest.raises(C.CtError) as e:
        C.ct_geom_create(C.geom_desc(get_config("c1")["geom"]), 0)
    assert e.value.status in (C.CT_E_CUDA, C.CT_E_CONFIG)


def test_invalid_geometry_rejected_before_device(C):
    from synth.configs import get_config
    g = dict(get_config("c1")["geom"], dx=-1.0)
    with pytest.raises(C.CtError) as e:
        C.ct_geom_create(C.geom_desc(g), 0)
    assert e.value.status == C.CT_E_CONFIG

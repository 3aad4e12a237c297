"""CPU-only checks of the product: the C-ABI library loads and exports every
declared symbol, and the host-side logic (problem construction, dof numbering,
Dirichlet sets) agrees with the oracle. No kernel is launched here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2509_17494_b200 as hb
from paper_2509_17494_b200 import _lib
from oracle import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols():
    hdr = open(os.path.join(ROOT, "include", "helmtg_b200.h")).read()
    declared = set(re.findall(r"\b(htg_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTS)
    L = C.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name


def test_config_default_matches_reference():  # proj/core/include/helmtg/twogrid.hpp:18-30
    cfg = _lib.Config()
    _lib.lib().htg_config_default(C.byref(cfg))
    d = hb.SolverConfig()
    for f, _ in _lib.Config._fields_:
        assert getattr(cfg, f) == getattr(d, f), f


@pytest.mark.parametrize("spec", [
    dict(order=4, wavelengths=20, ppw=10),
    dict(order=2, wavelengths=10, ppw=10),
    dict(order=4, wavelengths=5, ppw=10, layer_sides=(po.LEFT, po.BOTTOM), side_tags=(1, 2, 1, 2),
         layer_width_dofs=12),
    dict(order=6, wavelengths=3, ppw=8, side_tags=(0, 2, 2, 1), damping_D=0.01),
    dict(order=4, wavelengths=3, ppw=10, layer_sides=(po.TOP,), side_tags=(2, 2, 2, 1), damping_D=0.05,
         layer_width_dofs=8),
])
def test_build_problem_matches_oracle(spec):
    o = po.Session(po.ProblemSpec(**spec))
    p = hb.build_problem(hb.ProblemSpec(**spec))
    k, eps = o.coeffs()
    assert p.n_cells == o.nx
    assert np.array_equal(k, p.k_cells)
    assert np.allclose(eps, p.eps_cells, rtol=2e-16, atol=0)
    assert np.array_equal(o.rhs(), p.rhs)


@pytest.mark.parametrize("p", [2, 4, 6, 8])
def test_dof_numbering_matches_oracle(p):
    n = 3
    o = po.Session(desc=dict(order=p, nx=n, ny=n, h=1 / n, k=1.0, side_tags=(2, 2, 2, 2)))
    keys = o.dof_keys()
    kind, x, y, off = keys.T
    jx = np.where(kind == ord("h"), off + 1, np.where(kind == ord("c"), off // (p - 1) + 1, 0))
    jy = np.where(kind == ord("e"), off + 1, np.where(kind == ord("c"), off % (p - 1) + 1, 0))
    idx = hb.dof_index(n, n, p, x * p + jx, y * p + jy)
    assert np.array_equal(idx, np.arange(o.ndof))


def test_dirichlet_mask_matches_oracle():
    for tags in [(0, 2, 2, 2), (0, 0, 1, 2), (2, 1, 0, 0)]:
        o = po.Session(po.ProblemSpec(order=4, wavelengths=3, ppw=10, side_tags=tags))
        m = hb.dirichlet_mask(o.nx, o.ny, 4, tags)
        assert np.array_equal(np.flatnonzero(m), o.dirichlet_dofs())


def test_invalid_order_rejected():
    with pytest.raises(hb.HtgError) as e:
        hb.build_problem(hb.ProblemSpec(order=3, wavelengths=5, ppw=10))
    assert e.value.code == _lib.HTG_ERR_INVALID

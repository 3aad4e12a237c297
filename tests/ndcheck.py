"""ctypes driver for tests/native/libndcheck.so (test infrastructure): host-side
factor + solve of the coarse nested-dissection LU and its backward error."""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "native", "libndcheck.so")


def _lib():
    if not os.path.exists(LIB):
        import subprocess
        subprocess.run(["make", "-C", os.path.join(HERE, "..", "paper_2509_17494_b200", "csrc"), "ndcheck"],
                       check=True, capture_output=True)
    return C.CDLL(LIB)


def _cproblem(problem):
    from paper_2509_17494_b200 import _lib as hl
    k = np.ascontiguousarray(problem.k_cells, dtype=np.float64)
    e = np.ascontiguousarray(problem.eps_cells, dtype=np.float64)
    n = problem.n_cells
    cp = hl.Problem(problem.order, n, problem.ny or n, problem.h, problem.k, 0.0,
                    k.ctypes.data_as(C.POINTER(C.c_double)), e.ctypes.data_as(C.POINTER(C.c_double)),
                    (C.c_int * 4)(*problem.side_tags), None, None, None, None, int(problem.element_kind))
    return cp, (k, e)


def coarse_check(problem, rc, leaf=16, pivtol=0.1):
    """Solve A_c x = rc on the host with the ND factors; returns (x, backward error, stats)."""
    L = _lib()
    cp, keep = _cproblem(problem)
    nv = rc.shape[-1]
    a9 = np.zeros(nv * 9, np.complex128)
    assert L.nd_stencil(C.byref(cp), a9.ctypes.data_as(C.c_void_p), C.c_longlong(a9.size)) == 0
    rc = np.ascontiguousarray(np.atleast_2d(rc), dtype=np.complex128)
    x = np.zeros_like(rc)
    st = np.zeros(4)
    rcode = L.nd_check(C.byref(cp), int(leaf), C.c_double(pivtol), rc.ctypes.data_as(C.c_void_p),
                       x.ctypes.data_as(C.c_void_p), int(rc.shape[0]), st.ctypes.data_as(C.c_void_p))
    assert rcode == 0
    CX = int(round(np.sqrt(nv))) - 1
    A = a9.reshape(CX + 1, CX + 1, 3, 3)
    be = []
    for r in range(rc.shape[0]):
        X = np.pad(x[r].reshape(CX + 1, CX + 1), 1)
        y = np.zeros((CX + 1, CX + 1), np.complex128)
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                y += A[:, :, dy + 1, dx + 1] * X[1 + dy:CX + 2 + dy, 1 + dx:CX + 2 + dx]
        be.append(np.linalg.norm(y.ravel() - rc[r]) / np.linalg.norm(rc[r]))
    stats = dict(delayed=int(st[0]), max_front=int(st[1]), nodes=int(st[2]), shared=int(st[3]))
    return x, max(be), stats


def fe_apply(problem, q, alpha, x):
    """y = A x with the product's order-q FE lattice matrix (csrc/coarse_nd.cpp fe_lattice)."""
    L = _lib()
    cp, keep = _cproblem(problem)
    x = np.ascontiguousarray(x, dtype=np.complex128)
    y = np.zeros_like(x)
    assert L.nd_fe_apply(C.byref(cp), int(q), C.c_double(alpha), x.ctypes.data_as(C.c_void_p),
                         y.ctypes.data_as(C.c_void_p)) == 0
    return y


def fe_solve(problem, q, alpha, b, leaf=16, pivtol=0.3):
    """Solve A x = b with the ND factors of the order-q FE lattice matrix; returns (x, stats)."""
    L = _lib()
    cp, keep = _cproblem(problem)
    b = np.ascontiguousarray(np.atleast_2d(b), dtype=np.complex128)
    x = np.zeros_like(b)
    st = np.zeros(4)
    assert L.nd_check_fe(C.byref(cp), int(q), C.c_double(alpha), int(leaf), C.c_double(pivtol),
                         b.ctypes.data_as(C.c_void_p), x.ctypes.data_as(C.c_void_p), int(b.shape[0]),
                         st.ctypes.data_as(C.c_void_p)) == 0
    return x, dict(delayed=int(st[0]), max_front=int(st[1]), nodes=int(st[2]))

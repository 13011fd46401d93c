"""ORACLE (test infrastructure): ctypes wrappers for sf_oracle.c.

All arrays are float64 numpy.  Volume layout (nz, ny, nx); projections
(views, nt, ns).  Definitions: SURVEY.md 8c.1 (projector), Eq. 35
(regulariser).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force=False):
    """Compile the oracle with gcc -O2 -fopenmp (no fast-math)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + ".tmp%d" % os.getpid()
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                           "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _LIB)
    return _LIB


class OGeom(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double),
                ("ox", ctypes.c_double), ("oy", ctypes.c_double), ("oz", ctypes.c_double),
                ("arc", ctypes.c_int), ("ns", ctypes.c_int), ("nt", ctypes.c_int),
                ("ds", ctypes.c_double), ("dt", ctypes.c_double), ("off_s", ctypes.c_double),
                ("off_t", ctypes.c_double), ("dso", ctypes.c_double), ("dsd", ctypes.c_double),
                ("na", ctypes.c_int),
                ("orbit_deg", ctypes.c_double), ("orbit_start_deg", ctypes.c_double),
                ("pitch", ctypes.c_double), ("source_z0", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        d = ctypes.c_double
        i = ctypes.c_int
        _lib.og_forward.argtypes = [P(OGeom), P(d), i, i, i, P(d)]
        _lib.og_back.argtypes = [P(OGeom), P(d), i, i, i, P(d)]
        _lib.og_forward_rays.argtypes = [P(OGeom), P(d), i, P(i), P(i), P(i), P(d)]
        _lib.og_back_voxels.argtypes = [P(OGeom), P(d), i, i, i, i, P(ctypes.c_int64), P(d)]
        _lib.og_reg.argtypes = [P(OGeom), i, d, d, i, P(d), i, P(d), ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p]
        _lib.og_reg.restype = d
        _lib.og_reg_at.argtypes = [P(OGeom), i, d, d, i, P(d), i, P(d), ctypes.c_void_p, i,
                                   P(ctypes.c_int64), P(d), P(d)]
        _lib.og_directions.argtypes = [P(i)]
        _lib.og_set_threads.argtypes = [i]
        _lib.og_max_threads.restype = i
    return _lib


def set_threads(n):
    lib().og_set_threads(int(n))


def max_threads():
    return lib().og_max_threads()


def ogeom(g):
    """Oracle geometry struct from a synth geometry dict."""
    if int(g["ns"]) > 4096:
        raise ValueError("oracle supports ns <= 4096 (per-column F1 scratch)")
    return OGeom(int(g["dim"]), int(g["nx"]), int(g["ny"]), int(g["nz"] if g["dim"] == 3 else 1),
                 g["dx"], g["dy"], g["dz"], g["offset_x"], g["offset_y"], g["offset_z"],
                 1 if g["det"] == "arc" else 0, int(g["ns"]), int(g["nt"] if g["dim"] == 3 else 1),
                 g["ds"], g["dt"], g["offset_s"], g["offset_t"], g["dso"], g["dsd"], int(g["na"]),
                 g["orbit_deg"], g["orbit_start_deg"], g["pitch"], g["source_z0"])


def _p(a, ct=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def vol_shape(g):
    return (g["nz"] if g["dim"] == 3 else 1, g["ny"], g["nx"])


def proj_shape(g, count):
    return (count, g["nt"] if g["dim"] == 3 else 1, g["ns"])


def _views(g, views):
    if views is None:
        return (0, 1, g["na"])
    return tuple(int(v) for v in views)


def forward(g, x, views=None):
    """A x for the views (start, stride, count); x (nz, ny, nx)."""
    st, sd, cnt = _views(g, views)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(vol_shape(g))
    out = np.zeros(proj_shape(g, cnt), dtype=np.float64)
    G = ogeom(g)
    lib().og_forward(ctypes.byref(G), _p(x), st, sd, cnt, _p(out))
    return out


def back(g, proj, views=None):
    """A' proj for the views (start, stride, count)."""
    st, sd, cnt = _views(g, views)
    proj = np.ascontiguousarray(proj, dtype=np.float64).reshape(proj_shape(g, cnt))
    out = np.zeros(vol_shape(g), dtype=np.float64)
    G = ogeom(g)
    lib().og_back(ctypes.byref(G), _p(proj), st, sd, cnt, _p(out))
    return out


def forward_rays(g, x, v, s, t):
    """[A x] at individual rays (absolute view v, column s, row t)."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(vol_shape(g))
    v = np.ascontiguousarray(v, dtype=np.int32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    t = np.ascontiguousarray(t, dtype=np.int32)
    out = np.zeros(v.size, dtype=np.float64)
    G = ogeom(g)
    lib().og_forward_rays(ctypes.byref(G), _p(x), v.size, _p(v, ctypes.c_int), _p(s, ctypes.c_int),
                          _p(t, ctypes.c_int), _p(out))
    return out


def back_voxels(g, proj, views, idx):
    """[A' proj] at flat voxel indices idx (views = (start, stride, count))."""
    st, sd, cnt = _views(g, views)
    proj = np.ascontiguousarray(proj, dtype=np.float64).reshape(proj_shape(g, cnt))
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.zeros(idx.size, dtype=np.float64)
    G = ogeom(g)
    lib().og_back_voxels(ctypes.byref(G), _p(proj), st, sd, cnt, idx.size,
                         _p(idx, ctypes.c_int64), _p(out))
    return out


POTENTIALS = {"quadratic": 0, "hyperbola": 1, "fair": 2, "qggmrf": 3}
CURVATURES = {"huber": 0, "max": 1}


def _betas13(betas):
    b = np.zeros(13, dtype=np.float64)
    bb = np.asarray(betas, dtype=np.float64).ravel()[:13]
    b[:bb.size] = bb
    return b


def directions():
    arr = (ctypes.c_int * 39)()
    lib().og_directions(arr)
    return [tuple(arr[3 * d:3 * d + 3]) for d in range(13)]


def reg(g, potential, delta, betas, n_dirs, x, kappa=None, want_grad=True, want_curv=True, q=1.2,
        curvature="huber"):
    """Return (R(x), grad, curv) of Eq. 35 with the Huber curvature (x2 SQS split), or the
    maximum curvature (curvature="max"); q is the q-GGMRF exponent (potential "qggmrf")."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(vol_shape(g))
    b = _betas13(betas)
    grad = np.zeros_like(x) if want_grad else None
    curv = np.zeros_like(x) if want_curv else None
    kap = None
    if kappa is not None:
        kap = np.ascontiguousarray(kappa, dtype=np.float64).reshape(vol_shape(g))
    G = ogeom(g)
    val = lib().og_reg(ctypes.byref(G), POTENTIALS[potential], float(delta), float(q), CURVATURES[curvature],
                       _p(b), int(n_dirs), _p(x),
                       kap.ctypes.data if kap is not None else None,
                       grad.ctypes.data if grad is not None else None,
                       curv.ctypes.data if curv is not None else None)
    return val, grad, curv


def reg_at(g, potential, delta, betas, n_dirs, x, idx, kappa=None, q=1.2, curvature="huber"):
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(vol_shape(g))
    b = _betas13(betas)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    grad = np.zeros(idx.size)
    curv = np.zeros(idx.size)
    kap = None
    if kappa is not None:
        kap = np.ascontiguousarray(kappa, dtype=np.float64).reshape(vol_shape(g))
    G = ogeom(g)
    lib().og_reg_at(ctypes.byref(G), POTENTIALS[potential], float(delta), float(q), CURVATURES[curvature],
                    _p(b), int(n_dirs), _p(x),
                    kap.ctypes.data if kap is not None else None, idx.size, _p(idx, ctypes.c_int64),
                    _p(grad), _p(curv))
    return grad, curv

"""Thin ctypes binding of libctrecon.so (include/ctrecon.h) — marshalling only.

Every function has the C name and forwards device pointers of torch CUDA
tensors; no arithmetic of the method happens here.  If the shared library is
missing or was built for another GPU the import fails loudly: there is no CPU
fallback.
"""
import ctypes
import math
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libctrecon.so")   # scripts/kbench.py --lib points it at a tuning variant

CT_OK, CT_E_SHAPE, CT_E_CONFIG, CT_E_NUMERIC, CT_E_DIVERGED, CT_E_CUDA, CT_E_NCCL, CT_E_NOMEM = range(8)
STATUS_NAMES = ["CT_OK", "CT_E_SHAPE", "CT_E_CONFIG", "CT_E_NUMERIC", "CT_E_DIVERGED", "CT_E_CUDA",
                "CT_E_NCCL", "CT_E_NOMEM"]
CT_DET_FLAT, CT_DET_ARC = 0, 1
CT_POT = {"quadratic": 0, "hyperbola": 1, "fair": 2, "qggmrf": 3}
CT_CURV = {"huber": 0, "max": 1}
RHO_CONTINUATION, RHO_FIXED = 0, 1
PROPOSED, SIMPLE = 0, 1   # oslalm_variant: Algorithm 1 / Algorithm 2
INIT_LAST_SUBSET, INIT_FULL = 0, 1


class CtError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS_NAMES[status] if 0 <= status < 8 else status, msg))
        self.status = status


class ct_geom_desc(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double),
                ("offset_x", ctypes.c_double), ("offset_y", ctypes.c_double), ("offset_z", ctypes.c_double),
                ("det_shape", ctypes.c_int32), ("ns", ctypes.c_int32), ("nt", ctypes.c_int32),
                ("ds", ctypes.c_double), ("dt", ctypes.c_double),
                ("offset_s", ctypes.c_double), ("offset_t", ctypes.c_double),
                ("dso", ctypes.c_double), ("dsd", ctypes.c_double),
                ("na", ctypes.c_int32),
                ("orbit_deg", ctypes.c_double), ("orbit_start_deg", ctypes.c_double),
                ("pitch", ctypes.c_double), ("source_z0", ctypes.c_double)]


class ct_views(ctypes.Structure):
    _fields_ = [("start", ctypes.c_int32), ("stride", ctypes.c_int32), ("count", ctypes.c_int32)]


class ct_reg_desc(ctypes.Structure):
    _fields_ = [("potential", ctypes.c_int32), ("delta", ctypes.c_double), ("n_dirs", ctypes.c_int32),
                ("beta", ctypes.c_double * 13), ("curvature", ctypes.c_int32), ("q", ctypes.c_double)]


class oslalm_params(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int32), ("alpha", ctypes.c_double), ("rho_mode", ctypes.c_int32),
                ("rho_fixed", ctypes.c_double), ("init_grad", ctypes.c_int32),
                ("box_lo", ctypes.c_double), ("box_hi", ctypes.c_double), ("variant", ctypes.c_int32)]


class oslalm_state(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("g", ctypes.c_void_p), ("htilde", ctypes.c_void_p),
                ("k", ctypes.c_int64)]


EXPORTS = ["ct_geom_create", "ct_geom_destroy", "ct_forward", "ct_back", "ct_sqs_diag", "ct_kappa_weights", "ct_fbp",
           "ct_reg_grad",
           "oslalm_workspace_size", "oslalm_relaxed_solve", "oslalm_state_h", "oslalm_rho", "ct_sync",
           "ct_nccl_unique_id", "ct_dist_create", "ct_dist_destroy", "ct_launch_count", "ct_last_error",
           "oslalm_profile", "ct_count_nnz", "ct_zslab_range", "oslalm_zslab_workspace_size", "ct_sqs_diag_zslab",
           "oslalm_zslab_solve", "ct_sino_upload", "ct_count_work", "ct_zprefix_size", "ct_forward_zprefix",
           "oslalm_residual", "ct_dist_create_local", "ct_geom_set_fwd_segments", "ct_geom_fwd_segments"]

_lib = None


def load():
    """Load libctrecon.so (raises if it is absent: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError("libctrecon.so is not built (run `python -c 'import __graft_entry__ as g; g.build()'`)")
    L = ctypes.CDLL(LIB_PATH)
    P, vp, i32, f, st = ctypes.POINTER, ctypes.c_void_p, ctypes.c_int32, ctypes.c_float, ctypes.c_int
    L.ct_geom_create.argtypes = [P(ct_geom_desc), ctypes.c_int, P(vp)]
    L.ct_geom_destroy.argtypes = [vp]
    L.ct_geom_destroy.restype = None
    L.ct_forward.argtypes = [vp, vp, ct_views, vp, vp]
    L.ct_back.argtypes = [vp, vp, ct_views, f, ctypes.c_int, vp, vp]
    L.ct_zprefix_size.argtypes = [vp, P(ctypes.c_size_t)]
    L.ct_forward_zprefix.argtypes = [vp, vp, ct_views, vp, vp, ctypes.c_size_t, vp]
    L.ct_geom_set_fwd_segments.argtypes = [vp, ctypes.c_int]
    L.ct_geom_fwd_segments.argtypes = [vp, ctypes.c_int, P(ctypes.c_int)]
    L.oslalm_residual.argtypes = [vp, P(oslalm_params), vp, ctypes.c_int64, vp, ctypes.c_size_t, vp, vp]
    L.ct_sqs_diag.argtypes = [vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
    L.ct_reg_grad.argtypes = [vp, P(ct_reg_desc), vp, vp, vp, vp, vp]
    L.ct_kappa_weights.argtypes = [vp, vp, vp, vp, ctypes.c_size_t, vp]
    L.ct_fbp.argtypes = [vp, vp, vp, vp, ctypes.c_size_t, vp]
    L.ct_zslab_range.argtypes = [vp, ctypes.c_int, ctypes.c_int, P(ctypes.c_int), P(ctypes.c_int)]
    L.oslalm_zslab_workspace_size.argtypes = [vp, P(oslalm_params), ctypes.c_int, ctypes.c_int, P(ctypes.c_size_t)]
    L.ct_sqs_diag_zslab.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, vp, P(vp), P(vp), ctypes.c_size_t, vp]
    L.oslalm_zslab_solve.argtypes = [vp, vp, vp, P(ct_reg_desc), P(vp), P(oslalm_params), P(oslalm_state),
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, P(vp), ctypes.c_size_t, vp]
    L.oslalm_workspace_size.argtypes = [vp, P(oslalm_params), vp, P(ctypes.c_size_t)]
    L.oslalm_relaxed_solve.argtypes = [vp, vp, vp, P(ct_reg_desc), vp, vp, P(oslalm_params), P(oslalm_state),
                                       ctypes.c_int, vp, P(ctypes.c_double), vp, vp, ctypes.c_size_t, vp]
    L.oslalm_state_h.argtypes = [vp, vp, P(oslalm_state), vp, vp]
    L.oslalm_profile.argtypes = [vp, vp, vp, P(ct_reg_desc), vp, vp, P(oslalm_params), P(oslalm_state),
                                 ctypes.c_int, vp, vp, ctypes.c_size_t, vp, P(ctypes.c_double)]
    L.ct_count_nnz.argtypes = [vp, ct_views, vp, vp]
    L.ct_count_work.argtypes = [vp, ct_views, vp, vp]
    L.oslalm_rho.argtypes = [ctypes.c_int64, ctypes.c_double]
    L.oslalm_rho.restype = ctypes.c_double
    L.ct_sync.argtypes = [vp]
    L.ct_sino_upload.argtypes = [vp, vp, ct_views, vp, vp]
    L.ct_nccl_unique_id.argtypes = [P(ctypes.c_ubyte)]
    L.ct_dist_create.argtypes = [ctypes.c_int, ctypes.c_int, P(ctypes.c_ubyte), ctypes.c_int, P(vp)]
    L.ct_dist_create_local.argtypes = [ctypes.c_int, ctypes.c_int, P(vp)]
    L.ct_dist_destroy.argtypes = [vp]
    L.ct_dist_destroy.restype = None
    L.ct_launch_count.restype = ctypes.c_int64
    L.ct_last_error.restype = ctypes.c_char_p
    for name in ("ct_geom_create", "ct_forward", "ct_back", "ct_sqs_diag", "ct_kappa_weights", "ct_fbp", "ct_reg_grad",
                 "oslalm_workspace_size",
                 "oslalm_relaxed_solve", "oslalm_state_h", "ct_sync", "ct_nccl_unique_id", "ct_dist_create",
                 "oslalm_profile", "ct_count_nnz", "ct_zslab_range", "oslalm_zslab_workspace_size",
                 "ct_sqs_diag_zslab", "oslalm_zslab_solve", "ct_sino_upload", "ct_count_work", "ct_zprefix_size",
                 "ct_forward_zprefix", "oslalm_residual", "ct_dist_create_local", "ct_geom_set_fwd_segments",
                 "ct_geom_fwd_segments"):
        getattr(L, name).restype = st
    _lib = L
    return L


def _check(status):
    if status != CT_OK:
        raise CtError(status, load().ct_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if t.dtype != torch.float32 or not t.is_contiguous():
        raise ValueError("expected a contiguous float32 tensor")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


# ----------------------------------------------------------------- descriptors
def geom_desc(g):
    """ct_geom_desc from a geometry dict (keys as in synth/configs.py)."""
    return ct_geom_desc(int(g["dim"]), int(g["nx"]), int(g["ny"]), int(g["nz"] if g["dim"] == 3 else 1),
                        g["dx"], g["dy"], g["dz"], g["offset_x"], g["offset_y"], g["offset_z"],
                        CT_DET_ARC if g["det"] == "arc" else CT_DET_FLAT, int(g["ns"]),
                        int(g["nt"] if g["dim"] == 3 else 1), g["ds"], g["dt"], g["offset_s"], g["offset_t"],
                        g["dso"], g["dsd"], int(g["na"]), g["orbit_deg"], g["orbit_start_deg"], g["pitch"],
                        g["source_z0"])


def reg_desc(potential, delta, betas, n_dirs, curvature="huber", q=1.2):
    r = ct_reg_desc()
    r.potential = CT_POT[potential]
    r.delta = float(delta)
    r.curvature = CT_CURV[curvature]
    r.q = float(q)
    r.n_dirs = int(n_dirs)
    for i in range(13):
        r.beta[i] = float(betas[i]) if i < len(betas) else 0.0
    return r


def params(M, alpha, rho_mode=RHO_CONTINUATION, rho_fixed=0.0, init_grad=INIT_LAST_SUBSET, box_lo=0.0,
           box_hi=math.inf, variant=PROPOSED):
    return oslalm_params(int(M), float(alpha), int(rho_mode), float(rho_fixed), int(init_grad), float(box_lo),
                         float(box_hi), int(variant))


def views(start, stride, count):
    return ct_views(int(start), int(stride), int(count))


# ----------------------------------------------------------------- functions
def ct_geom_create(desc, device=0):
    h = ctypes.c_void_p()
    _check(load().ct_geom_create(ctypes.byref(desc), int(device), ctypes.byref(h)))
    return h


def ct_geom_destroy(h):
    load().ct_geom_destroy(h)


def ct_forward(geom, x, v, proj, stream=None):
    _check(load().ct_forward(geom, _ptr(x), v, _ptr(proj), _stream(stream)))


def ct_zprefix_size(geom):
    n = ctypes.c_size_t()
    _check(load().ct_zprefix_size(geom, ctypes.byref(n)))
    return n.value


def ct_forward_zprefix(geom, x, v, proj, workspace, stream=None):
    _check(load().ct_forward_zprefix(geom, _ptr(x), v, _ptr(proj), ctypes.c_void_p(workspace.data_ptr()),
                                     workspace.numel() * workspace.element_size(), _stream(stream)))


def ct_geom_set_fwd_segments(geom, nseg):
    _check(load().ct_geom_set_fwd_segments(geom, int(nseg)))


def ct_geom_fwd_segments(geom, views=128):
    """Segments the z-prefix forward uses for a launch of `views` views (0 = unsegmented)."""
    n = ctypes.c_int()
    _check(load().ct_geom_fwd_segments(geom, int(views), ctypes.byref(n)))
    return n.value


def oslalm_residual(geom, p, k, workspace, r_out, dist=None, stream=None):
    _check(load().oslalm_residual(geom, ctypes.byref(p), dist, int(k), ctypes.c_void_p(workspace.data_ptr()),
                                  workspace.numel() * workspace.element_size(), _ptr(r_out), _stream(stream)))


def ct_back(geom, proj, v, x_out, scale=1.0, accumulate=False, stream=None):
    _check(load().ct_back(geom, _ptr(proj), v, float(scale), int(bool(accumulate)), _ptr(x_out), _stream(stream)))


def ct_sqs_diag(geom, w, d_out, workspace, dist=None, stream=None):
    _check(load().ct_sqs_diag(geom, _ptr(w), dist, _ptr(d_out), ctypes.c_void_p(workspace.data_ptr()),
                              workspace.numel() * workspace.element_size(), _stream(stream)))


def ct_fbp(geom, proj, x_out, workspace, stream=None):
    _check(load().ct_fbp(geom, _ptr(proj), _ptr(x_out), ctypes.c_void_p(workspace.data_ptr()),
                         workspace.numel() * workspace.element_size(), _stream(stream)))


def ct_kappa_weights(geom, w, kappa_out, workspace, stream=None):
    _check(load().ct_kappa_weights(geom, _ptr(w), _ptr(kappa_out), ctypes.c_void_p(workspace.data_ptr()),
                                   workspace.numel() * workspace.element_size(), _stream(stream)))


def ct_reg_grad(geom, reg, x, grad, curv=None, kappa=None, stream=None):
    _check(load().ct_reg_grad(geom, ctypes.byref(reg), _ptr(x), _ptr(kappa), _ptr(grad), _ptr(curv),
                              _stream(stream)))


def oslalm_workspace_size(geom, p, dist=None):
    n = ctypes.c_size_t()
    _check(load().oslalm_workspace_size(geom, ctypes.byref(p), dist, ctypes.byref(n)))
    return n.value


def make_state(x, g, htilde, k=0):
    return oslalm_state(_ptr(x).value, _ptr(g).value, _ptr(htilde).value, int(k))


def oslalm_relaxed_solve(geom, y, w, reg, kappa, d_l, p, state, n_subiters, workspace, x_ref=None,
                         rms_per_iter=None, dist=None, stream=None):
    rms = None
    if rms_per_iter is not None:
        rms = (ctypes.c_double * max(1, len(rms_per_iter)))()
    _check(load().oslalm_relaxed_solve(geom, _ptr(y), _ptr(w), ctypes.byref(reg), _ptr(kappa), _ptr(d_l),
                                       ctypes.byref(p), ctypes.byref(state), int(n_subiters), _ptr(x_ref), rms,
                                       dist, ctypes.c_void_p(workspace.data_ptr()),
                                       workspace.numel() * workspace.element_size(), _stream(stream)))
    if rms is not None:
        for i in range(len(rms_per_iter)):
            rms_per_iter[i] = rms[i]
    return state


def oslalm_profile(geom, y, w, reg, kappa, d_l, p, state, n_subiters, workspace, dist=None, stream=None):
    """Returns summed device ms of [update, forward+residual, back+epilogue, rest]."""
    ms = (ctypes.c_double * 4)()
    _check(load().oslalm_profile(geom, _ptr(y), _ptr(w), ctypes.byref(reg), _ptr(kappa), _ptr(d_l),
                                 ctypes.byref(p), ctypes.byref(state), int(n_subiters), dist,
                                 ctypes.c_void_p(workspace.data_ptr()), workspace.numel() * workspace.element_size(),
                                 _stream(stream), ms))
    return [ms[i] for i in range(4)]


def ct_count_nnz(geom, v, stream=None):
    """Number of nonzero entries of A on views v (device count, returned as int)."""
    cnt = torch.zeros(1, dtype=torch.int64, device=torch.device("cuda", torch.cuda.current_device()))
    _check(load().ct_count_nnz(geom, v, ctypes.c_void_p(cnt.data_ptr()), _stream(stream)))
    return int(cnt.item())


def ct_count_work(geom, v, stream=None):
    """(nnz, in-cone voxel-view pairs, in-cone column-view pairs) of A on views v."""
    cnt = torch.zeros(3, dtype=torch.int64, device=torch.device("cuda", torch.cuda.current_device()))
    _check(load().ct_count_work(geom, v, ctypes.c_void_p(cnt.data_ptr()), _stream(stream)))
    return tuple(int(c) for c in cnt.tolist())


def oslalm_state_h(geom, d_l, state, h_out, stream=None):
    _check(load().oslalm_state_h(geom, _ptr(d_l), ctypes.byref(state), _ptr(h_out), _stream(stream)))


def oslalm_rho(k, alpha):
    return load().oslalm_rho(int(k), float(alpha))


def ct_sino_upload(geom, host, v, dev, stream=None):
    """Copy views v of a (na, nt, ns) float32 host array (pinned) into the same rows of dev."""
    if host.is_cuda or host.dtype != torch.float32 or not host.is_contiguous():
        raise ValueError("host must be a contiguous float32 CPU tensor")
    if host.shape != dev.shape:
        raise ValueError("host and device sinograms differ in shape")
    _check(load().ct_sino_upload(geom, ctypes.c_void_p(host.data_ptr()), v, _ptr(dev), _stream(stream)))


def ct_sync(stream=None):
    _check(load().ct_sync(_stream(stream)))


def ct_nccl_unique_id():
    buf = (ctypes.c_ubyte * 128)()
    _check(load().ct_nccl_unique_id(buf))
    return bytes(buf)


def ct_dist_create(rank, world, uid, device):
    buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
    h = ctypes.c_void_p()
    _check(load().ct_dist_create(int(rank), int(world), buf, int(device), ctypes.byref(h)))
    return h


def ct_dist_create_local(world, device=0):
    """Single-process emulation of a `world`-rank view-sharded solve on one device."""
    h = ctypes.c_void_p()
    _check(load().ct_dist_create_local(int(world), int(device), ctypes.byref(h)))
    return h


def ct_dist_destroy(h):
    load().ct_dist_destroy(h)


def ct_launch_count():
    return load().ct_launch_count()


# ----------------------------------------------------------------- z-slab decomposition
def ct_zslab_range(geom, rank, world):
    z0, nz = ctypes.c_int(), ctypes.c_int()
    _check(load().ct_zslab_range(geom, int(rank), int(world), ctypes.byref(z0), ctypes.byref(nz)))
    return z0.value, nz.value


def oslalm_zslab_workspace_size(geom, p, rank, world):
    n = ctypes.c_size_t()
    _check(load().oslalm_zslab_workspace_size(geom, ctypes.byref(p), int(rank), int(world), ctypes.byref(n)))
    return n.value


def _ptr_array(ts):
    return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def ct_sqs_diag_zslab(geom, w, d_outs, workspaces, world, dist=None, stream=None):
    nbytes = min(t.numel() * t.element_size() for t in workspaces)
    _check(load().ct_sqs_diag_zslab(geom, _ptr(w), len(d_outs), int(world), dist, _ptr_array(d_outs),
                                    _ptr_array(workspaces), nbytes, _stream(stream)))


def oslalm_zslab_solve(geom, y, w, reg, d_ls, p, states, n_subiters, workspaces, world, dist=None, stream=None):
    """states: a list of oslalm_state (one per local slab); their k is advanced."""
    arr = (oslalm_state * len(states))(*states)
    nbytes = min(t.numel() * t.element_size() for t in workspaces)
    _check(load().oslalm_zslab_solve(geom, _ptr(y), _ptr(w), ctypes.byref(reg), _ptr_array(d_ls), ctypes.byref(p),
                                     arr, len(states), int(world), int(n_subiters), dist, _ptr_array(workspaces),
                                     nbytes, _stream(stream)))
    for i, s_ in enumerate(states):
        s_.k = arr[i].k

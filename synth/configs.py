"""The five BASELINE.json configs as plain numbers.

Geometry keys mirror `ct_geom_desc` in include/ctrecon.h (lengths in mm,
angles in degrees).  Where BASELINE.json leaves a number open the value is
the SURVEY.md section 8d choice (GE-LightSpeed-class detector pitch and
offsets, Dso 541 / Dsd 949, helix centred on the volume); DESIGN.md lists
every such reading.

Regulariser (Eq. 35): 13 directions in 3-D (26 neighbours,
PAPER.md:321), 4 in 2-D (8 neighbours); beta_i = beta0 * w_i with
w_i = dx / |physical offset of direction i|.  beta0 per
config was chosen once by `scripts/calibrate_beta.py`, which calls only
`oracle/` (beta0 = 0.05 * median(D_L) / (4 * sum_i w_i)).
"""
import copy
import math

# Direction offsets (ox, oy, oz) in voxel units; the first four are the
# in-plane ones used in 2-D.  Every unordered neighbour pair appears once.
DIRECTIONS = [
    (1, 0, 0), (0, 1, 0), (1, 1, 0), (1, -1, 0),
    (0, 0, 1), (1, 0, 1), (-1, 0, 1), (0, 1, 1), (0, -1, 1),
    (1, 1, 1), (-1, 1, 1), (1, -1, 1), (-1, -1, 1),
]


def _helical_z0(na, nt, dt, dso, dsd, pitch, orbit_deg, offset_z=0.0):
    """source_z0 that centres the helix on the volume."""
    table_per_turn = pitch * nt * dt * dso / dsd
    zstep = table_per_turn * (orbit_deg / 360.0) / na
    return offset_z - 0.5 * (na - 1) * zstep


def _geom(**kw):
    g = dict(dim=3, nx=1, ny=1, nz=1, dx=1.0, dy=1.0, dz=1.0,
             offset_x=0.0, offset_y=0.0, offset_z=0.0,
             det="arc", ns=1, nt=1, ds=1.0, dt=1.0, offset_s=0.0, offset_t=0.0,
             dso=541.0, dsd=949.0, na=1, orbit_deg=360.0, orbit_start_deg=0.0,
             pitch=0.0, source_z0=0.0)
    g.update(kw)
    return g


CONFIGS = {
    # BASELINE.json configs[0]: 2-D fan, 128^2 @ 1.0 mm, 256 bins, 180 views.
    "c1": dict(
        geom=_geom(dim=2, nx=128, ny=128, nz=1, dx=1.0, dy=1.0, dz=1.0,
                   det="arc", ns=256, nt=1, ds=1.266, offset_s=0.25, na=180),
        phantom=dict(seed=1001, n_ellipsoids=10),
        noise=dict(seed=2001, I0=1e4, sigma=0.0),
        reg=dict(potential="hyperbola", delta=0.01, n_dirs=4, beta0=None),
        solver=dict(M=4, iters=20, alpha=1.999),
    ),
    # configs[1]: 2-D fan, 512^2 @ 0.98 mm, 888 bins, 984 views.
    "c2": dict(
        geom=_geom(dim=2, nx=512, ny=512, nz=1, dx=0.98, dy=0.98, dz=1.0,
                   det="arc", ns=888, nt=1, ds=1.0239, offset_s=1.25, na=984),
        phantom=dict(seed=1002, n_ellipsoids=10),
        noise=dict(seed=2002, I0=1e5, sigma=5.0),
        reg=dict(potential="hyperbola", delta=0.01, n_dirs=4, beta0=None),
        solver=dict(M=41, iters=30, alpha=1.999),
    ),
    # configs[2]: 3-D axial cone, flat 444x32, 256^2x64 @ 1 mm, 492 views.
    "c3": dict(
        geom=_geom(dim=3, nx=256, ny=256, nz=64, dx=1.0, dy=1.0, dz=1.0,
                   det="flat", ns=444, nt=32, ds=1.532, dt=3.508, offset_s=0.25,
                   na=492),
        phantom=dict(seed=1003, n_ellipsoids=12),
        noise=dict(seed=2003, I0=1e5, sigma=0.0),
        reg=dict(potential="hyperbola", delta=0.01, n_dirs=13, beta0=None),
        solver=dict(M=12, iters=30, alpha=1.999),
    ),
    # configs[3]: 3-D helical, arc 888x64, 512^2x96 @ 0.98/0.625, 3 turns.
    "c4": dict(
        geom=_geom(dim=3, nx=512, ny=512, nz=96, dx=0.98, dy=0.98, dz=0.625,
                   det="arc", ns=888, nt=64, ds=1.0239, dt=1.0964, offset_s=1.25,
                   na=2952, orbit_deg=1080.0, pitch=1.0,
                   source_z0=_helical_z0(2952, 64, 1.0964, 541.0, 949.0, 1.0, 1080.0)),
        phantom=dict(seed=1004, n_ellipsoids=16),
        noise=dict(seed=2004, I0=5e4, sigma=5.0),
        reg=dict(potential="hyperbola", delta=0.01, n_dirs=13, beta0=None),
        solver=dict(M=24, iters=30, alpha=1.999),
    ),
    # configs[4]: as c4 at 1024^2x256 @ 0.49/0.625, 6 turns.
    "c5": dict(
        geom=_geom(dim=3, nx=1024, ny=1024, nz=256, dx=0.49, dy=0.49, dz=0.625,
                   det="arc", ns=888, nt=64, ds=1.0239, dt=1.0964, offset_s=1.25,
                   na=5904, orbit_deg=2160.0, pitch=1.0,
                   source_z0=_helical_z0(5904, 64, 1.0964, 541.0, 949.0, 1.0, 2160.0)),
        phantom=dict(seed=1005, n_ellipsoids=32),
        noise=dict(seed=2005, I0=2e4, sigma=0.0),
        reg=dict(potential="hyperbola", delta=0.01, n_dirs=13, beta0=None),
        solver=dict(M=41, iters=20, alpha=1.999),
    ),
}

# beta0 written by scripts/calibrate_beta.py (oracle-only); see module doc.
_BETA0 = {"c1": 3.744e5, "c2": 4.539e7, "c3": 3.278e6, "c4": 1.512e7, "c5": 1.746e6}


def get_config(name):
    cfg = copy.deepcopy(CONFIGS[name])
    if cfg["reg"]["beta0"] is None and _BETA0.get(name) is not None:
        cfg["reg"]["beta0"] = _BETA0[name]
    return cfg


def reg_directions(n_dirs):
    return DIRECTIONS[:n_dirs]


def reg_betas(geom, beta0, n_dirs):
    """beta_i = beta0 * dx / |offset_i| in mm (13 entries, zeros past n_dirs)."""
    out = [0.0] * 13
    for i, (ox, oy, oz) in enumerate(DIRECTIONS[:n_dirs]):
        dist = math.sqrt((ox * geom["dx"]) ** 2 + (oy * geom["dy"]) ** 2 + (oz * geom["dz"]) ** 2)
        out[i] = beta0 * geom["dx"] / dist
    return out


def subset_views(na, M, m):
    """View descriptor (start, stride, count) of subset m: views v = m mod M
    (SURVEY.md 8c.3 #4)."""
    return (m, M, (na - m + M - 1) // M)


def shrink(cfg, nx=None, nz=None, na=None, ns=None, nt=None):
    """A smaller copy of a config with the same geometry family (for tests)."""
    c = copy.deepcopy(cfg)
    g = c["geom"]
    if nx is not None:
        scale = g["nx"] / nx
        g["nx"] = g["ny"] = nx
        g["dx"] *= scale
        g["dy"] *= scale
    if nz is not None and g["dim"] == 3:
        g["dz"] *= g["nz"] / nz
        g["nz"] = nz
    if ns is not None:
        g["ds"] *= g["ns"] / ns
        g["offset_s"] = g["offset_s"] * ns / g["ns"]
        g["ns"] = ns
    if nt is not None and g["dim"] == 3:
        g["dt"] *= g["nt"] / nt
        g["nt"] = nt
    if na is not None:
        turns = g["orbit_deg"] / 360.0
        g["na"] = na
        if g["pitch"] != 0.0:
            g["source_z0"] = _helical_z0(na, g["nt"], g["dt"], g["dso"], g["dsd"],
                                         g["pitch"], g["orbit_deg"], g["offset_z"])
        del turns
    return c


def shard_views(na, M, m, rank, world):
    """Rank `rank` of `world` takes the subset-local views rank, rank+world, ...
    of subset m: (m + rank*M, world*M, ceil((V_m - rank)/world)) — the same rule
    as the device-side view selection of libctrecon."""
    vm = (na - m + M - 1) // M
    return (m + rank * M, world * M, max(0, (vm - rank + world - 1) // world))

"""Seeded random ellipse/ellipsoid phantoms, their voxelisation and their
analytic line integrals (SURVEY.md 8d "Phantom generator", 8c.5 chord formula).

Everything here is float64 torch so it runs on the CPU (tests) or on a GPU
(bench inputs at c4/c5 sizes) with the same code.  Random numbers are drawn
with numpy PCG64 from the config seed, so the ellipsoid list is identical on
every device.
"""
import math

import numpy as np
import torch


def sample_ellipsoids(geom, n_ellipsoids, seed, max_tries=1000):
    """Body + (n-1) disjoint inserts inside the body.

    Returns an (n, 8) float64 array: cx, cy, cz, ax, ay, az, angle, density.
    Angles rotate about z only.  2-D configs use az = inf-like (ignored).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    W = geom["nx"] * geom["dx"]
    Z = geom["nz"] * geom["dz"]
    three_d = geom["dim"] == 3
    oz = geom["offset_z"]
    body = [
        geom["offset_x"] + rng.uniform(-0.02, 0.02) * W,
        geom["offset_y"] + rng.uniform(-0.02, 0.02) * W,
        oz,
        rng.uniform(0.38, 0.45) * W,
        rng.uniform(0.30, 0.40) * W,
        0.45 * Z if three_d else 1.0,
        rng.uniform(0.0, math.pi),
        0.02,
    ]
    ells = [body]
    bx, by, bz, ba, bb, bc, bang, _ = body
    cb, sb = math.cos(bang), math.sin(bang)

    def inside_body(px, py, pz):
        u = (px - bx) * cb + (py - by) * sb
        v = -(px - bx) * sb + (py - by) * cb
        r = (u / ba) ** 2 + (v / bb) ** 2
        if three_d:
            r += ((pz - bz) / bc) ** 2
        return r < 1.0

    spheres = []  # bounding spheres of accepted inserts
    tries = 0
    while len(ells) < n_ellipsoids and tries < max_tries:
        tries += 1
        # centre uniform inside 70% of the body
        while True:
            u, v = rng.uniform(-1, 1, size=2)
            w = rng.uniform(-1, 1) if three_d else 0.0
            if u * u + v * v + w * w < 1.0:
                break
        u, v, w = 0.7 * u * ba, 0.7 * v * bb, 0.7 * w * bc
        cx = bx + u * cb - v * sb
        cy = by + u * sb + v * cb
        cz = bz + w if three_d else oz
        ax = rng.uniform(0.03, 0.12) * W
        ay = rng.uniform(0.03, 0.12) * W
        az = rng.uniform(0.05, 0.2) * Z if three_d else 1.0
        ang = rng.uniform(0.0, math.pi)
        dens = rng.uniform(-0.02, 0.02)
        r = max(ax, ay, az) if three_d else max(ax, ay)
        # bounding sphere inside the body: sample its surface
        ok = True
        for th in np.linspace(0, 2 * math.pi, 24, endpoint=False):
            for ph in (np.linspace(-math.pi / 2, math.pi / 2, 9) if three_d else [0.0]):
                px = cx + r * math.cos(ph) * math.cos(th)
                py = cy + r * math.cos(ph) * math.sin(th)
                pz = cz + r * math.sin(ph)
                if not inside_body(px, py, pz):
                    ok = False
                    break
            if not ok:
                break
        if not ok:
            continue
        if three_d and (cz - r < oz - Z / 2 or cz + r > oz + Z / 2):
            continue
        for (sx, sy, sz, sr) in spheres:
            if (sx - cx) ** 2 + (sy - cy) ** 2 + (sz - cz) ** 2 < (sr + r) ** 2:
                ok = False
                break
        if not ok:
            continue
        spheres.append((cx, cy, cz, r))
        ells.append([cx, cy, cz, ax, ay, az, ang, dens])
    return np.array(ells, dtype=np.float64)


def voxelize(geom, ells, sub=None, device="cpu"):
    """Voxel averages of the phantom with sub^d sub-samples per voxel.

    Returns a float64 tensor (nz, ny, nx) (nz = 1 in 2-D).  Vectorised over
    ellipsoids and blocks of z-slices."""
    three_d = geom["dim"] == 3
    if sub is None:
        sub = 4 if not three_d else 2
    nx, ny, nz = geom["nx"], geom["ny"], geom["nz"] if three_d else 1
    dx, dy, dz = geom["dx"], geom["dy"], geom["dz"]
    f = torch.float64
    e = torch.as_tensor(np.asarray(ells, dtype=np.float64), device=device)
    cx, cy, cz, ax, ay, az, ang, dens = e.unbind(1)
    c, s = torch.cos(ang), torch.sin(ang)
    xc = (torch.arange(nx, dtype=f, device=device) - (nx - 1) / 2) * dx + geom["offset_x"]
    yc = (torch.arange(ny, dtype=f, device=device) - (ny - 1) / 2) * dy + geom["offset_y"]
    zc = (torch.arange(nz, dtype=f, device=device) - (nz - 1) / 2) * dz + geom["offset_z"]
    offs = [((i + 0.5) / sub - 0.5) for i in range(sub)]
    zoffs = offs if three_d else [0.0]
    out = torch.zeros((nz, ny, nx), dtype=f, device=device)
    zb = max(1, int(32e6 // max(1, ny * nx * len(ells))))
    for k0 in range(0, nz, zb):
        k1 = min(nz, k0 + zb)
        acc = torch.zeros((k1 - k0, ny, nx), dtype=f, device=device)
        for oz_ in zoffs:
            Z = (zc[k0:k1] + oz_ * dz)[:, None, None, None]
            for oy_ in offs:
                Y = (yc + oy_ * dy)[None, :, None, None]
                for ox_ in offs:
                    X = (xc + ox_ * dx)[None, None, :, None]
                    u = (X - cx) * c + (Y - cy) * s
                    v = -(X - cx) * s + (Y - cy) * c
                    r = (u / ax) ** 2 + (v / ay) ** 2
                    if three_d:
                        r = r + ((Z - cz) / az) ** 2
                    acc += ((r <= 1.0).to(f) * dens).sum(-1)
        out[k0:k1] = acc / (sub ** (3 if three_d else 2))
    return out


def line_integrals(ells, P, D, three_d):
    """Sum of ellipsoid chords along rays P + lambda*D (|D| = 1), SURVEY 8c.5.

    P, D: (..., 3) float64 tensors.  Returns (...) float64.  Vectorised over
    the ellipsoids (one set of tensor ops for all of them)."""
    e = torch.as_tensor(np.asarray(ells, dtype=np.float64), device=P.device)
    cx, cy, cz, ax, ay, az, ang, dens = e.unbind(1)
    c, s = torch.cos(ang), torch.sin(ang)
    px = P[..., 0:1] - cx
    py = P[..., 1:2] - cy
    pu = (px * c + py * s) / ax
    pv = (-px * s + py * c) / ay
    du = (D[..., 0:1] * c + D[..., 1:2] * s) / ax
    dv = (-D[..., 0:1] * s + D[..., 1:2] * c) / ay
    dd = du * du + dv * dv
    pd = pu * du + pv * dv
    pp = pu * pu + pv * pv
    if three_d:
        pw = (P[..., 2:3] - cz) / az
        dw = D[..., 2:3] / az
        dd = dd + dw * dw
        pd = pd + pw * dw
        pp = pp + pw * pw
    disc = pd * pd - dd * (pp - 1.0)
    return (dens * 2.0 * torch.sqrt(torch.clamp(disc, min=0.0)) / dd).sum(-1)


def view_angles(geom, views):
    """beta_v (rad) and source z for view indices (tensor, float64)."""
    na = geom["na"]
    beta = math.radians(geom["orbit_start_deg"]) + math.radians(geom["orbit_deg"]) * views / na
    table = geom["pitch"] * geom["nt"] * geom["dt"] * geom["dso"] / geom["dsd"]
    zstep = table * (geom["orbit_deg"] / 360.0) / na
    zs = geom["source_z0"] + views * zstep
    return beta, zs


def rays(geom, views, s_pos, t_pos):
    """Source points and unit directions for detector positions.

    views: (V,) float64 view indices; s_pos: (ns',) fractional column
    indices; t_pos: (nt',) fractional row indices.  Returns P, D with shape
    (V, nt', ns', 3).  Cell centres are at integer indices."""
    dev = views.device
    f = torch.float64
    beta, zs = view_angles(geom, views)
    cb, sb = torch.cos(beta)[:, None, None], torch.sin(beta)[:, None, None]
    ns, nt = geom["ns"], geom["nt"]
    arc = geom["det"] == "arc"
    delta = geom["ds"] / geom["dsd"] if arc else geom["ds"]
    sig = ((s_pos - (ns - 1) / 2 - geom["offset_s"]) * delta)[None, None, :]
    if geom["dim"] == 3:
        th = ((t_pos - (nt - 1) / 2 - geom["offset_t"]) * geom["dt"])[None, :, None]
    else:
        th = torch.zeros((1, t_pos.numel(), 1), dtype=f, device=dev)
    dso, dsd = geom["dso"], geom["dsd"]
    Sx, Sy = dso * cb, dso * sb
    ecx, ecy = -cb, -sb
    eux, euy = -sb, cb
    if arc:
        dx_ = dsd * (torch.cos(sig) * ecx + torch.sin(sig) * eux)
        dy_ = dsd * (torch.cos(sig) * ecy + torch.sin(sig) * euy)
    else:
        dx_ = dsd * ecx + sig * eux
        dy_ = dsd * ecy + sig * euy
    shape = (views.numel(), t_pos.numel(), s_pos.numel())
    dx_ = dx_.expand(shape)
    dy_ = dy_.expand(shape)
    dz_ = th.expand(shape)
    n = torch.sqrt(dx_ * dx_ + dy_ * dy_ + dz_ * dz_)
    D = torch.stack([dx_ / n, dy_ / n, dz_ / n], dim=-1)
    P = torch.stack([Sx.expand(shape), Sy.expand(shape),
                     zs[:, None, None].expand(shape)], dim=-1)
    return P, D


def analytic_sinogram(geom, ells, views=None, sub_s=2, sub_t=2, device="cpu", chunk=None):
    """Analytic line integrals averaged over sub_s x sub_t sub-rays per cell.

    Returns float64 (V, nt, ns) (nt = 1 in 2-D)."""
    f = torch.float64
    if views is None:
        views = torch.arange(geom["na"], dtype=f, device=device)
    three_d = geom["dim"] == 3
    ns = geom["ns"]
    nt = geom["nt"] if three_d else 1
    if not three_d:
        sub_t = 1
    so = (torch.arange(sub_s, dtype=f, device=device) + 0.5) / sub_s - 0.5
    to = (torch.arange(sub_t, dtype=f, device=device) + 0.5) / sub_t - 0.5
    scol = torch.arange(ns, dtype=f, device=device)
    trow = torch.arange(nt, dtype=f, device=device)
    out = torch.zeros((views.numel(), nt, ns), dtype=f, device=device)
    if chunk is None:   # keep the (views, rows, cols, ellipsoids) temporaries near 64 M elements
        chunk = max(1, int(64e6 // max(1, nt * ns * len(ells))))
    for v0 in range(0, views.numel(), chunk):
        vv = views[v0:v0 + chunk]
        acc = torch.zeros((vv.numel(), nt, ns), dtype=f, device=device)
        for a in so:
            for b in to:
                P, D = rays(geom, vv, scol + a, trow + b if three_d else trow)
                acc += line_integrals(ells, P, D, three_d)
        out[v0:v0 + chunk] = acc / (sub_s * sub_t)
    return out

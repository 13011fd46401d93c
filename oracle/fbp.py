"""ORACLE (test infrastructure): filtered back-projection initialiser, float64.

PAPER.md:334 starts Algorithm 1 from "an initial (FBP) image" (SURVEY.md 8f
row f3).  The paper does not define its FBP; this is the textbook fan-beam
FBP (Kak & Slaney, "Principles of Computerized Tomographic Imaging", ch. 3.4:
equiangular and equispaced fan beams) and its Feldkamp (FDK) cone-beam
extension for axial scans, written out step by step:

  virtual detector through the isocentre (D = Dso):
    flat: s = sigma * D/Dsd (mm), rows t = theta * D/Dsd
    arc : gamma = sigma (radians), rows t = theta * D/Dsd
  1. pre-weight   flat: R' = R D / sqrt(D^2 + s^2 + t^2)
                  arc : R' = R D cos(gamma) D / sqrt(D^2 + t^2)
  2. filter each row with the band-limited ramp of the sampling interval
     (Ram-Lak): Q = (1/2) Delta sum_k R'_k h[n - k],
       h[0] = 1/(4 Delta^2), h[odd m] = -1/(m^2 pi^2 Delta^2) (flat),
       h[odd m] = -1/(pi^2 sin^2(m Delta)) (arc: (m D/sin)^2 scaling), else 0
  3. back-project every voxel P with linear interpolation on the detector:
     a = (P-S).e_c, b = (P-S).e_u, L = |P-S|_xy,
       flat: s' = D b / a, t' = D (z - z_s)/a, weight (D/a)^2
       arc : gamma' = atan2(b, a), t' = D (z - z_s)/L, weight 1/L^2
     f(P) = (2 pi / na) sum_v weight Q_v(s', t')      (full 360 degree orbit)
Supported: 2-D fan and 3-D axial (pitch 0) with a 360 degree orbit.
Only tests/, smoke() and bench.py's cpu_baseline may import this module.
"""
import math

import numpy as np

from . import projector as P


def supported(g):
    return abs(g["orbit_deg"] - 360.0) < 1e-9 and (g["dim"] == 2 or g["pitch"] == 0.0)


def ramp_kernel(ns, delta, arc):
    """h[m], m = -(ns-1) .. ns-1 (Ram-Lak, sampling interval delta)."""
    m = np.arange(-(ns - 1), ns)
    h = np.zeros(m.size)
    h[m == 0] = 1.0 / (4.0 * delta * delta)
    odd = (m % 2) != 0
    if arc:
        h[odd] = -1.0 / (math.pi ** 2 * np.sin(m[odd] * delta) ** 2)
    else:
        h[odd] = -1.0 / (math.pi ** 2 * (m[odd] * delta) ** 2)
    return h


def fbp(g, proj):
    """FBP / FDK image (nz, ny, nx) from line integrals proj (na, nt, ns)."""
    if not supported(g):
        raise ValueError("FBP needs a 360-degree 2-D fan or axial cone scan")
    three_d = g["dim"] == 3
    ns, na = g["ns"], g["na"]
    nt = g["nt"] if three_d else 1
    arc = g["det"] == "arc"
    D, Dsd = g["dso"], g["dsd"]
    proj = np.asarray(proj, dtype=np.float64).reshape(na, nt, ns)
    delta = g["ds"] / Dsd if arc else g["ds"]
    sig = (np.arange(ns) - (ns - 1) / 2.0 - g["offset_s"]) * delta
    th = (np.arange(nt) - (nt - 1) / 2.0 - g["offset_t"]) * g["dt"] if three_d else np.zeros(1)
    tv = th * D / Dsd                                   # rows on the virtual detector (mm)
    if arc:
        dv = delta                                      # filter sampling: angle
        w = D * np.cos(sig)[None, :] * (D / np.sqrt(D * D + tv * tv))[:, None]
    else:
        sv = sig * D / Dsd
        dv = delta * D / Dsd                            # filter sampling: mm at the isocentre
        w = D / np.sqrt(D * D + sv[None, :] ** 2 + tv[:, None] ** 2)
    h = ramp_kernel(ns, dv, arc)
    # 1-2: pre-weight and filter every row (full convolution, centre ns samples)
    q = np.empty_like(proj)
    for v in range(na):
        for t in range(nt):
            q[v, t] = 0.5 * dv * np.convolve(proj[v, t] * w[t], h)[ns - 1:2 * ns - 1]
    # 3: voxel-driven back-projection with bilinear interpolation
    nz, ny, nx = P.vol_shape(g)
    xs = (np.arange(nx) - (nx - 1) / 2.0) * g["dx"] + g["offset_x"]
    ys = (np.arange(ny) - (ny - 1) / 2.0) * g["dy"] + g["offset_y"]
    zs = (np.arange(nz) - (nz - 1) / 2.0) * g["dz"] + g["offset_z"]
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    out = np.zeros((nz, ny, nx))
    s_c0 = (ns - 1) / 2.0 + g["offset_s"]
    t_c0 = (nt - 1) / 2.0 + g["offset_t"]
    for v in range(na):
        beta = math.radians(g["orbit_start_deg"]) + 2.0 * math.pi * v / na
        cb, sb = math.cos(beta), math.sin(beta)
        zsrc = g["source_z0"] if three_d else 0.0
        rx, ry = X - D * cb, Y - D * sb
        a = -(rx * cb + ry * sb)
        b = ry * cb - rx * sb
        if arc:
            L2 = rx * rx + ry * ry
            ucol = np.arctan2(b, a) / delta + s_c0
            tt = D * (Z - zsrc) / np.sqrt(L2)
            wgt = 1.0 / L2
        else:
            ucol = (D * b / a) / (delta * D / Dsd) + s_c0
            tt = D * (Z - zsrc) / a
            wgt = (D / a) ** 2
        urow = tt / (g["dt"] * D / Dsd) + t_c0 if three_d else np.zeros_like(ucol)
        out += wgt * _interp2(q[v], urow, ucol)
    return out * (2.0 * math.pi / na)


def _interp2(img, r, c):
    """Bilinear interpolation of img (nt, ns) at fractional (row, col); 0 outside."""
    nt, ns = img.shape
    c0 = np.floor(c).astype(np.int64)
    fc = c - c0
    if nt == 1:
        r0 = np.zeros_like(c0)
        fr = np.zeros_like(c)
    else:
        r0 = np.floor(r).astype(np.int64)
        fr = r - r0
    val = np.zeros_like(c)
    for dr, wr in ((0, 1.0 - fr), (1, fr)):
        for dc, wc in ((0, 1.0 - fc), (1, fc)):
            rr, cc = r0 + dr, c0 + dc
            ok = (rr >= 0) & (rr < nt) & (cc >= 0) & (cc < ns)
            val += np.where(ok, wr * wc * img[np.clip(rr, 0, nt - 1), np.clip(cc, 0, ns - 1)], 0.0)
    return val

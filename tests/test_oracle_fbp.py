"""Pins of the oracle FBP/FDK initialiser (oracle/fbp.py).

Textbook facts, not the oracle's own formula: FBP of the exact line integrals
of a uniform disk (2-D fan, arc and flat) reproduces the density inside the
disk and the error falls under refinement; FDK is exact on the mid-plane of an
axial scan for a z-invariant object; the reconstruction rotates with the
sinogram (rot90 when the views are rolled by na/4)."""
import math

import numpy as np
import pytest

from oracle import fbp as F
from synth.configs import _geom
from synth.phantom import analytic_sinogram


def disk_geom(det, n, ns_scale=1):
    ds = 1.266 if det == "arc" else 1.4
    return _geom(dim=2, nx=n, ny=n, nz=1, dx=64.0 / n, dy=64.0 / n, det=det, ns=int(72 * ns_scale * n / 32),
                 ds=ds * 32 / n / ns_scale, offset_s=0.25, dso=100.0, dsd=180.0, na=int(120 * n / 32))


def disk(g, r, mu):
    return np.array([[0.0, 0.0, 0.0, r, r, 1.0, 0.0, mu]])


def interior_err(g, img, r, mu, frac=0.6):
    n = g["nx"]
    xs = (np.arange(n) - (n - 1) / 2.0) * g["dx"]
    X, Y = np.meshgrid(xs, xs)
    m = X ** 2 + Y ** 2 < (frac * r) ** 2
    return np.sqrt(np.mean((img[0][m] - mu) ** 2)) / mu


@pytest.mark.parametrize("det", ["arc", "flat"])
def test_fbp_uniform_disk_and_refinement(det):
    errs = []
    for n in (32, 64):
        g = disk_geom(det, n)
        mu, r = 0.02, 20.0
        sino = analytic_sinogram(g, disk(g, r, mu), sub_s=1).numpy()
        img = F.fbp(g, sino)
        errs.append(interior_err(g, img, r, mu))
    assert errs[0] < 2e-3, errs          # 2.4e-4 (arc) / 5.8e-4 (flat) at n = 32
    assert errs[1] < 0.6 * errs[0], errs


@pytest.mark.parametrize("det", ["arc", "flat"])
def test_fdk_midplane_of_z_invariant_object(det):
    # a long cylinder (ellipsoid with a huge z semi-axis): axial FDK is exact on the mid-plane
    g = _geom(dim=3, nx=48, ny=48, nz=5, dx=1.3, dy=1.3, dz=1.0, det=det, ns=120, nt=12,
              ds=1.266 if det == "arc" else 1.4, dt=1.6, offset_s=0.25, offset_t=0.0, dso=100.0, dsd=180.0,
              na=240)
    mu, r = 0.02, 20.0
    ell = np.array([[0.0, 0.0, 0.0, r, r, 1e4, 0.0, mu]])
    sino = analytic_sinogram(g, ell, sub_s=1, sub_t=1).numpy()
    img = F.fbp(g, sino)
    n = g["nx"]
    xs = (np.arange(n) - (n - 1) / 2.0) * g["dx"]
    X, Y = np.meshgrid(xs, xs)
    m = X ** 2 + Y ** 2 < (0.6 * r) ** 2
    mid = img[2][m]
    assert np.sqrt(np.mean((mid - mu) ** 2)) / mu < 0.03


def test_fbp_rotates_with_the_sinogram():
    g = disk_geom("arc", 32)
    g["na"] = 120
    rng = np.random.default_rng(1)
    ells = np.array([[4.0, -3.0, 0.0, 9.0, 5.0, 1.0, 0.4, 0.02], [-6.0, 5.0, 0.0, 4.0, 3.0, 1.0, 1.1, 0.01]])
    sino = analytic_sinogram(g, ells, sub_s=1).numpy() + 1e-4 * rng.standard_normal((g["na"], 1, g["ns"]))
    g0 = dict(g, offset_s=0.0)
    a = F.fbp(g0, sino)
    b = F.fbp(g0, np.roll(sino, -g["na"] // 4, axis=0))
    # rolling the views by a quarter turn rotates the image by 90 degrees about the centre
    assert np.allclose(b[0], np.rot90(a[0], k=1), atol=1e-12) or np.allclose(b[0], np.rot90(a[0], k=-1), atol=1e-12)


def test_fbp_rejects_helical():
    g = _geom(dim=3, nx=8, ny=8, nz=4, det="arc", ns=20, nt=4, na=10, pitch=1.0)
    with pytest.raises(ValueError):
        F.fbp(g, np.zeros((10, 4, 20)))

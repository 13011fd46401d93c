"""Noisy sinogram, statistical weights and initial image for a config.

Data model (BASELINE.json configs):
    l      = analytic line integrals of the phantom (cell-averaged sub-rays)
    c      = Poisson(I0 * exp(-l)) + N(0, sigma^2)
    c~     = max(c, 1)
    y      = log(I0 / c~),   w = c~          ("W = counts")
Initial image x0: the paper starts from an FBP image; FBP is
out of this round's scope, so x0 is the voxelised phantom blurred by a
Gaussian (sigma 1.5 voxels in-plane, 1 voxel in z) - a smooth, FBP-like
starting point that needs no reconstruction arithmetic (DESIGN.md reading).
"""
import math

import torch

from .phantom import analytic_sinogram, sample_ellipsoids, voxelize


def _gauss_blur(vol, sig_xy=1.5, sig_z=1.0):
    f = vol.dtype

    def kern(sig):
        r = int(math.ceil(3 * sig))
        xs = torch.arange(-r, r + 1, dtype=f, device=vol.device)
        k = torch.exp(-0.5 * (xs / sig) ** 2)
        return k / k.sum(), r

    out = vol
    nz, ny, nx = out.shape
    kx, r = kern(sig_xy)
    # along x
    o = out.reshape(-1, 1, nx)
    o = torch.nn.functional.conv1d(o, kx.view(1, 1, -1), padding=r)
    out = o.reshape(nz, ny, nx)
    # along y
    o = out.permute(0, 2, 1).reshape(-1, 1, ny)
    o = torch.nn.functional.conv1d(o, kx.view(1, 1, -1), padding=r)
    out = o.reshape(nz, nx, ny).permute(0, 2, 1)
    if nz > 1 and sig_z > 0:
        kz, rz = kern(sig_z)
        o = out.permute(1, 2, 0).reshape(-1, 1, nz)
        o = torch.nn.functional.conv1d(o, kz.view(1, 1, -1), padding=rz)
        out = o.reshape(ny, nx, nz).permute(2, 0, 1)
    return out.contiguous()


def make_dataset(cfg, device="cpu", sub_s=2, sub_t=2, vox_sub=None, with_truth=True):
    """Return dict with float64 tensors y, w (V, nt, ns); x_true, x0 (nz, ny, nx)."""
    g = cfg["geom"]
    ells = sample_ellipsoids(g, cfg["phantom"]["n_ellipsoids"], cfg["phantom"]["seed"])
    ell = analytic_sinogram(g, ells, sub_s=sub_s, sub_t=sub_t, device=device)
    gen = torch.Generator(device=device)
    gen.manual_seed(cfg["noise"]["seed"])
    I0 = cfg["noise"]["I0"]
    counts = torch.poisson(I0 * torch.exp(-ell), generator=gen)
    sigma = cfg["noise"]["sigma"]
    if sigma > 0:
        counts = counts + sigma * torch.randn(counts.shape, generator=gen, dtype=counts.dtype,
                                              device=device)
    ct = torch.clamp(counts, min=1.0)
    y = torch.log(I0 / ct)
    w = ct
    out = dict(y=y, w=w, ells=ells, ell=ell)
    if with_truth:
        xt = voxelize(g, ells, sub=vox_sub, device=device)
        out["x_true"] = xt
        out["x0"] = torch.clamp(_gauss_blur(xt), min=0.0)
    return out

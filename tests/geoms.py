"""Tiny geometries for CPU pins and GPU parity (same families as BASELINE configs)."""
import copy

from synth.configs import _geom, _helical_z0


def tiny(kind, **over):
    if kind == "fan2d_arc":
        g = _geom(dim=2, nx=16, ny=16, nz=1, dx=1.0, dy=1.0, det="arc", ns=32, ds=1.4,
                  offset_s=0.25, dso=100.0, dsd=180.0, na=24)
    elif kind == "fan2d_flat":
        g = _geom(dim=2, nx=16, ny=14, nz=1, dx=1.0, dy=1.1, offset_x=0.3, offset_y=-0.2,
                  det="flat", ns=36, ds=1.3, offset_s=-0.35, dso=100.0, dsd=180.0, na=20,
                  orbit_start_deg=7.0)
    elif kind == "axial_flat":
        g = _geom(dim=3, nx=12, ny=12, nz=8, dx=1.0, dy=1.0, dz=1.2, det="flat", ns=30, nt=14,
                  ds=1.5, dt=1.9, offset_s=0.25, offset_t=0.3, dso=100.0, dsd=180.0, na=18)
    elif kind == "helical_arc":
        g = _geom(dim=3, nx=12, ny=10, nz=10, dx=1.0, dy=1.0, dz=0.8, det="arc", ns=30, nt=8,
                  ds=1.5, dt=1.6, offset_s=1.25, offset_t=-0.2, dso=100.0, dsd=180.0, na=40,
                  orbit_deg=720.0, pitch=1.0)
        g["source_z0"] = _helical_z0(g["na"], g["nt"], g["dt"], g["dso"], g["dsd"], 1.0, 720.0)
    else:
        raise KeyError(kind)
    g.update(over)
    return copy.deepcopy(g)


KINDS = ["fan2d_arc", "fan2d_flat", "axial_flat", "helical_arc"]

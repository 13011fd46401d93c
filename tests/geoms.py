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
    elif kind == "helical_fine":
        # fine detector pitch: voxel footprints span 3..11 columns, so the GPU back-projector's
        # 4-, 6- and 8-column windows and its general (> 8 columns) loop all run
        g = _geom(dim=3, nx=12, ny=12, nz=9, dx=1.0, dy=1.0, dz=0.8, det="arc", ns=104, nt=10,
                  ds=0.3, dt=1.3, offset_s=0.75, offset_t=0.1, dso=100.0, dsd=180.0, na=30,
                  orbit_deg=720.0, pitch=0.8)
        g["source_z0"] = _helical_z0(g["na"], g["nt"], g["dt"], g["dso"], g["dsd"], 0.8, 720.0)
    elif kind == "axial_fine":
        g = _geom(dim=3, nx=10, ny=12, nz=6, dx=1.0, dy=0.9, dz=1.1, det="flat", ns=76, nt=12,
                  ds=0.45, dt=1.7, offset_s=-0.4, offset_t=0.2, dso=100.0, dsd=180.0, na=16,
                  orbit_start_deg=11.0)
    else:
        raise KeyError(kind)
    g.update(over)
    return copy.deepcopy(g)


KINDS = ["fan2d_arc", "fan2d_flat", "axial_flat", "helical_arc"]
FINE_KINDS = ["helical_fine", "axial_fine"]  # GPU parity only (wide-footprint code paths)


def mid(kind, **over):
    """Mid-size geometries that select the kernel instances the BASELINE 3-D configs
    run (the tiny ones above only reach the smallest):
      helical_mid   arc, nt = 64 (two rows per lane in the forward), 160 columns x 240
                    views per subset at M = 2 (>= 148 x 8 x 2 four-warp blocks: the 4-warp
                    forward in the solve), nz = 56 (three 24-voxel back-projector z-chunks,
                    the last ragged; two update z-chunks with the per-row prefix exchange),
                    H = 1.4-2.4 rows per voxel (24-voxel chunks span 34-58 rows: two
                    40-row passes in the back-projector)
      helical_rpl4  flat, nt = 96 (four rows per lane), 4-warp forward over all views, nz = 80
                    (four 24-voxel z-chunks, the last ragged: the back-projector's chunks share
                    each column's footprint)
      axial_mid     flat axial, nt = 40, nz = 50 (two update z-chunks)
      helical_thin  helical_mid with 12 planes: every hit spans <= 32 detector rows (one row
                    per lane in the z-prefix forward, as in thin z-slabs)"""
    if kind == "helical_mid":
        g = _geom(dim=3, nx=36, ny=36, nz=56, dx=1.0, dy=1.0, dz=1.0, det="arc", ns=160, nt=64,
                  ds=0.625, dt=1.0, offset_s=0.75, offset_t=-0.3, dso=100.0, dsd=180.0, na=480,
                  orbit_deg=720.0, pitch=1.0)
        g["source_z0"] = _helical_z0(g["na"], g["nt"], g["dt"], g["dso"], g["dsd"], 1.0, 720.0)
    elif kind == "helical_rpl4":
        g = _geom(dim=3, nx=32, ny=30, nz=80, dx=1.0, dy=1.0, dz=0.8, det="flat", ns=128, nt=96,
                  ds=0.7, dt=0.8, offset_s=-0.6, offset_t=0.4, dso=100.0, dsd=180.0, na=300,
                  orbit_deg=720.0, pitch=0.9, orbit_start_deg=5.0)
        g["source_z0"] = _helical_z0(g["na"], g["nt"], g["dt"], g["dso"], g["dsd"], 0.9, 720.0)
    elif kind == "helical_thin":
        # helical_mid cut to 12 planes: a voxel column spans 17-29 detector rows, so the z-prefix
        # forward takes one row per lane (the path of thin z-slabs)
        g = mid("helical_mid", nz=12, dz=1.0)
    elif kind == "axial_mid":
        g = _geom(dim=3, nx=40, ny=40, nz=50, dx=1.0, dy=1.0, dz=1.0, det="flat", ns=120, nt=40,
                  ds=0.95, dt=1.6, offset_s=0.25, offset_t=0.1, dso=110.0, dsd=200.0, na=240)
    else:
        raise KeyError(kind)
    g.update(over)
    return copy.deepcopy(g)


MID_KINDS = ["helical_mid", "helical_rpl4", "axial_mid", "helical_thin"]


def fwd3_blocks(g, count):
    """Grid of the 3-D forward (proj_fwd.cu fwd3_rpl): 4-warp blocks of 16 detector columns
    x views when that fills >= 2 waves of 8 blocks per SM on 148 SMs, else 2-warp blocks;
    rows per lane RPL = 1 / 2 / 4 for nt <= 32 / 64 / 128."""
    b4 = -(-g["ns"] // 16) * count
    nw = 4 if b4 >= 148 * 8 * 2 else 2
    rpl = 1 if g["nt"] <= 32 else 2 if g["nt"] <= 64 else 4
    return nw, rpl

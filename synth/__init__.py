"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package is the scanner simulator, not the method: it draws random
ellipse/ellipsoid phantoms, computes their analytic line integrals along
source-to-detector rays, adds Poisson/electronic noise and derives the
statistical weights.  It holds none of the reconstruction arithmetic
(no projector footprints, no regulariser, no Algorithm 1).  Both `oracle/`
and `paper_1512_04564_b200/` consume its arrays; neither is imported here.

Config numbers (geometry, M, alpha, iterations) follow BASELINE.json
`configs` and the choices of SURVEY.md section 8d; see DESIGN.md.
"""
from .configs import CONFIGS, get_config, reg_directions, reg_betas  # noqa: F401

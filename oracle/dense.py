"""ORACLE (test infrastructure): tiny dense-matrix forms of the method.

* `dense_A`           — the SF system matrix of a tiny geometry, column by
                        column from oracle.projector.forward.
* `literal_eq25`      — the literal proposed relaxed LALM, Eq. 25
                         with an explicit G^{1/2} from eigh,
                        quadratic loss g(u) = 1/2||u - y||^2 (after the Eq. 36
                        substitution A <- W^{1/2}A, y <- W^{1/2}y).
* `eq33`              — Eq. 33 on the same dense problem.
* `literal_eq18`      — LALM with simple relaxation, Eq. 18
                        with the relaxation variable of Eq. 10,
                        the same quadratic loss: the M = 1 form of Algorithm 2.
* `dense_pwls_quadratic` — the exact minimiser of Eq. 34 with a quadratic
                        potential, (A'WA + H_R)^{-1} A'W y, built from
                        finite-difference matrices C_i written out here.

Q_psi uses the caller's diagonal D_psi at x^(k) (Eq. 17); phi is the box
indicator of Omega = {x >= 0} whose prox on a separable quadratic is the clamp.
"""
import numpy as np

from . import projector as P


def dense_A(g, views=None):
    shape = P.vol_shape(g)
    n = int(np.prod(shape))
    cols = []
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        cols.append(P.forward(g, e.reshape(shape), views).ravel())
    return np.stack(cols, axis=1)


def sqrtm_psd(G, neg_tol=1e-8):
    lam, V = np.linalg.eigh(G)
    if lam.min() < -neg_tol * max(1.0, abs(lam).max()):
        raise ValueError("G = D_A - A'A is not PSD (min eig %g)" % lam.min())
    return (V * np.sqrt(np.clip(lam, 0.0, None))) @ V.T


def literal_eq25(A, y, DA, x0, alpha, rhos, psi_grad, psi_curv, lo=0.0):
    """Eq. 25 iterates (x_k, u_k, mu_k, v_k, nu_k) for k = 0..len(rhos).

    A, y are post-substitution (A <- W^{1/2}A, y <- W^{1/2}y).
    Initialisation (Theorem 2): u0 = A x0,
    mu0 = y - u0, v0 = G^{1/2} x0, nu0 = 0.
    """
    G = np.diag(DA) - A.T @ A
    Gh = sqrtm_psd(G)
    x = np.array(x0, dtype=np.float64)
    u = A @ x
    mu = y - u
    v = Gh @ x
    nu = np.zeros_like(v)
    xs, nus = [x.copy()], [nu.copy()]
    for rho in rhos:
        gp = psi_grad(x)
        Dp = psi_curv(x)
        # x-update: the quadratic part has Hessian rho A'A + rho G = rho D_A.
        rhs = Dp * x - gp + A.T @ mu + Gh @ nu + rho * (A.T @ u) + rho * (Gh @ v)
        x = np.maximum((rhs) / (Dp + rho * DA), lo)
        r_u = alpha * (A @ x) + (1.0 - alpha) * u
        u = (y - mu + rho * r_u) / (1.0 + rho)           # argmin 1/2||u-y||^2 + <mu,u> + rho/2||r_u-u||^2
        mu = mu - rho * (r_u - u)
        r_v = alpha * (Gh @ x) + (1.0 - alpha) * v
        v = r_v - nu / rho
        nu = nu - rho * (r_v - v)
        xs.append(x.copy())
        nus.append(nu.copy())
    return xs, nus


def literal_eq18(A, y, DA, x0, alpha, rhos, psi_grad, psi_curv, lo=0.0):
    """Eq. 18 iterates x_k for k = 0..len(rhos), written in (x, u, mu):
      x+ = argmin phi(x) + Q_psi(x; x) - <mu, Ax> + rho/2 ||Ax - u||^2 + rho/2 ||x - x_k||_G^2,
           G = D_A - A'A (Eq. 16): Hessian D_psi + rho D_A, so
           x+ = [ (D_psi x_k - grad psi + A'mu + rho A'u + rho G x_k) / (D_psi + rho D_A) ]_Omega;
      r  = alpha A x+ + (1 - alpha) u                                  (Eq. 10)
      u+ = argmin 1/2||u - y||^2 + <mu, u> + rho/2 ||r - u||^2 = (y - mu + rho r) / (1 + rho);
      mu+ = mu - rho (r - u+).
    Initialisation u0 = A x0, mu0 = y - u0 (then A'(u - y) is Algorithm 2's g)."""
    x = np.array(x0, dtype=np.float64)
    u = A @ x
    mu = y - u
    xs = [x.copy()]
    for rho in rhos:
        gp = psi_grad(x)
        Dp = psi_curv(x)
        Gx = DA * x - A.T @ (A @ x)
        x = np.maximum((Dp * x - gp + A.T @ mu + rho * (A.T @ u) + rho * Gx) / (Dp + rho * DA), lo)
        r = alpha * (A @ x) + (1.0 - alpha) * u
        u = (y - mu + rho * r) / (1.0 + rho)
        mu = mu - rho * (r - u)
        xs.append(x.copy())
    return xs


def eq33(A, y, DA, x0, alpha, rhos, psi_grad, psi_curv, lo=0.0):
    """Eq. 33 iterates with g0 = zeta0, h0 = D_A x0 - zeta0."""
    x = np.array(x0, dtype=np.float64)
    zeta = A.T @ (A @ x - y)
    g = zeta.copy()
    h = DA * x - zeta
    xs = [x.copy()]
    for rho in rhos:
        gamma = (rho - 1.0) * g + rho * h
        gp = psi_grad(x)
        Dp = psi_curv(x)
        x = np.maximum((Dp * x - gp + gamma) / (Dp + rho * DA), lo)
        zeta = A.T @ (A @ x - y)
        g = rho / (rho + 1.0) * (alpha * zeta + (1.0 - alpha) * g) + g / (rho + 1.0)
        h = alpha * (DA * x - zeta) + (1.0 - alpha) * h
        xs.append(x.copy())
    return xs


def diff_matrices(shape, dirs):
    """Finite-difference matrices C_i: [C_i x]_n = x_n - x_{n+s_i} for every
    in-bounds pair (n, n+s_i); one per direction offset (dx, dy, dz)."""
    nz, ny, nx = shape
    n = nz * ny * nx
    mats = []
    for (ox, oy, oz) in dirs:
        rows = []
        for k in range(nz):
            for j in range(ny):
                for i in range(nx):
                    i2, j2, k2 = i + ox, j + oy, k + oz
                    if 0 <= i2 < nx and 0 <= j2 < ny and 0 <= k2 < nz:
                        r = np.zeros(n)
                        r[(k * ny + j) * nx + i] = 1.0
                        r[(k2 * ny + j2) * nx + i2] = -1.0
                        rows.append(r)
        mats.append(np.array(rows).reshape(-1, n))
    return mats


def dense_pwls_quadratic(A, w, y, shape, dirs, betas):
    """argmin 1/2||y - Ax||_W^2 + sum_i beta_i sum_n 1/2 [C_i x]_n^2 (kappa = 1)."""
    H = A.T @ (w[:, None] * A)
    for C, b in zip(diff_matrices(shape, dirs), betas):
        if C.size:
            H = H + b * C.T @ C
    return np.linalg.solve(H, A.T @ (w * y))

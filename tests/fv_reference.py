"""Independent term-by-term finite-volume assembly of the Cartesian operator (test helper).

Deliberately shares no code path with the oracle or the library (the same role as the
reference's tests/oracles.hpp:46-105, which assembles the icosahedral operator directly from
profiles and geometry): every flux is written from the PDE
    -w^2 div_h(alpha_S grad_h u) - w^2 d_z(alpha_r d_z u) + beta u
integrated over the cell [x_i, x_i+hx] x [y_j, y_j+hy] x [z_k, z_k+1] with doubly periodic
horizontal boundaries and homogeneous Neumann top/bottom (flat geometry).
Rows/columns are in the reference's Field order: index = cell * nz + k (k fastest).
"""
import numpy as np
import scipy.sparse as sp


def assemble(P, level_scale: int = 1) -> sp.csr_matrix:
    nx, ny, nz = P.nx, P.ny, P.nz
    hx, hy = P.hx, P.hy
    z = P.z_faces
    w2 = P.omega * P.omega
    dz = np.diff(z)
    n = nx * ny * nz
    rows, cols, vals = [], [], []

    def idx(i, j, k):
        return ((j % ny) * nx + (i % nx)) * nz + k

    hT_b = P.beta_s.reshape(ny, nx)
    hT_a = P.alpha_r_s.reshape(ny, nx)
    se = P.alpha_s_s[: nx * ny].reshape(ny, nx)
    sn = P.alpha_s_s[nx * ny:].reshape(ny, nx)
    for j in range(ny):
        for i in range(nx):
            for k in range(nz):
                r = idx(i, j, k)
                diag = hx * hy * dz[k] * P.beta_r[k] * hT_b[j, i]
                # horizontal faces: coefficient w^2 alpha_S (face area) / (centre distance)
                for (ii, jj, coef) in (
                        (i + 1, j, w2 * P.alpha_s_r[k] * se[j, i] * dz[k] * hy / hx),
                        (i - 1, j, w2 * P.alpha_s_r[k] * se[j, (i - 1) % nx] * dz[k] * hy / hx),
                        (i, j + 1, w2 * P.alpha_s_r[k] * sn[j, i] * dz[k] * hx / hy),
                        (i, j - 1, w2 * P.alpha_s_r[k] * sn[(j - 1) % ny, i] * dz[k] * hx / hy)):
                    diag += coef
                    rows.append(r); cols.append(idx(ii, jj, k)); vals.append(-coef)
                # vertical faces k (below) and k+1 (above); Neumann: none at z_0 and z_nz
                for (kk, face) in ((k - 1, k), (k + 1, k + 1)):
                    if 0 <= kk < nz:
                        dist = 0.5 * (z[face + 1] - z[face - 1])
                        coef = w2 * P.alpha_r_r[face] * hT_a[j, i] * hx * hy / dist
                        diag += coef
                        rows.append(r); cols.append(idx(i, j, kk)); vals.append(-coef)
                rows.append(r); cols.append(r); vals.append(diag)
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))

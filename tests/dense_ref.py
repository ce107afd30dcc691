"""Independent dense reference for pinning the oracle (test helper, not the oracle).

Nothing here reuses the oracle's derivative matrix, geometric factors or
operator code: Lagrange-basis derivatives come from explicit polynomial
coefficients (numpy.polynomial), the Jacobian from the analytic derivatives of
the trilinear map through the element's 8 corner nodes, and the element
stiffness is the quadrature sum K_e[a,b] = sum_q W_q J_q grad(phi_a).grad(phi_b)
(SURVEY.md C-7 "dense assembly").  The GLL rule itself is pinned separately
(tests/test_oracle_gll.py), so taking nodes/weights from it is allowed here.
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import polynomial as P


def lagrange_deriv_matrix(nodes: np.ndarray) -> np.ndarray:
    """Dm[q, a] = l_a'(x_q) from the explicit coefficients of l_a."""
    n = len(nodes)
    Dm = np.zeros((n, n))
    for a in range(n):
        others = np.array([nodes[b] for b in range(n) if b != a])
        coef = P.polyfromroots(others) if len(others) else np.array([1.0])
        denom = np.prod(nodes[a] - others) if len(others) else 1.0
        Dm[:, a] = P.polyval(nodes, P.polyder(coef)) / denom
    return Dm


def element_corners(xyz: np.ndarray, e: int, n: int) -> np.ndarray:
    """corners[cz, cy, cx, :] = physical position of reference corner (+-1, +-1, +-1)."""
    n3 = n ** 3
    C = np.zeros((2, 2, 2, 3))
    for cz in range(2):
        for cy in range(2):
            for cx in range(2):
                q = (n - 1) * cx + n * (n - 1) * cy + n * n * (n - 1) * cz
                C[cz, cy, cx] = xyz[:, e * n3 + q]
    return C


def trilinear(C: np.ndarray, xi, eta, zeta):
    """Position and Jacobian d x_a / d xi_b of the trilinear map at one point."""
    N = lambda c, t: (1.0 - t) / 2.0 if c == 0 else (1.0 + t) / 2.0
    dN = lambda c, t: -0.5 if c == 0 else 0.5
    pos = np.zeros(3)
    J = np.zeros((3, 3))
    for cz in range(2):
        for cy in range(2):
            for cx in range(2):
                X = C[cz, cy, cx]
                pos += N(cx, xi) * N(cy, eta) * N(cz, zeta) * X
                J[:, 0] += dN(cx, xi) * N(cy, eta) * N(cz, zeta) * X
                J[:, 1] += N(cx, xi) * dN(cy, eta) * N(cz, zeta) * X
                J[:, 2] += N(cx, xi) * N(cy, eta) * dN(cz, zeta) * X
    return pos, J


def element_stiffness(C: np.ndarray, nodes: np.ndarray, weights: np.ndarray) -> np.ndarray:
    """K_e[a, b] with basis index a = i + n j + n^2 k (SURVEY.md C-4 local order)."""
    n = len(nodes)
    n3 = n ** 3
    Dm = lagrange_deriv_matrix(nodes)
    K = np.zeros((n3, n3))
    eye = np.eye(n)
    for qk in range(n):
        for qj in range(n):
            for qi in range(n):
                _, J = trilinear(C, nodes[qi], nodes[qj], nodes[qk])
                detJ = np.linalg.det(J)
                Jinv = np.linalg.inv(J)            # Jinv[b, a] = d xi_b / d x_a
                # reference gradients of all basis functions at this point
                gr = np.einsum("i,j,k->kji", Dm[qi], eye[qj], eye[qk]).reshape(n3)
                gs = np.einsum("i,j,k->kji", eye[qi], Dm[qj], eye[qk]).reshape(n3)
                gt = np.einsum("i,j,k->kji", eye[qi], eye[qj], Dm[qk]).reshape(n3)
                gref = np.stack([gr, gs, gt], axis=1)      # [n3, 3]
                gphys = gref @ Jinv                       # [n3, 3]
                W = weights[qi] * weights[qj] * weights[qk]
                K += W * detJ * (gphys @ gphys.T)
    return K


def assemble(mesh, nodes, weights):
    """Global stiffness K_G (n_global x n_global) and the element blocks."""
    geo = mesh.geom()
    gid, mask, _, _ = mesh.maps()
    n = mesh.n
    n3 = n ** 3
    KG = np.zeros((mesh.n_global, mesh.n_global))
    blocks = []
    for e in range(mesh.E):
        Ke = element_stiffness(element_corners(geo["xyz"], e, n), nodes, weights)
        blocks.append(Ke)
        g = gid[e * n3:(e + 1) * n3]
        KG[np.ix_(g, g)] += Ke
    return KG, blocks, gid, mask

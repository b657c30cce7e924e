"""ABCD-matrix algebra (oracle; test infrastructure only, see oracle/__init__.py).

Matrices are 4x4 real, row-major [[A, B], [C, D]] as in Eq. Intro04.
"""
import numpy as np

TAU_SYM = 1e-10  # validity tolerance (SPEC.md:32 tau_sym; reading R6)


def blocks(M):
    """Split a 4x4 ABCD matrix into its 2x2 blocks A, B, C, D (Eq. Intro04)."""
    M = np.asarray(M, dtype=np.float64)
    return M[0:2, 0:2], M[0:2, 2:4], M[2:4, 0:2], M[2:4, 2:4]


def assemble(A, B, C, D):
    return np.block([[A, B], [C, D]])


def residuals(M):
    """The three residuals of Eq. Intro12:
    AB^T - BA^T, CD^T - DC^T, AD^T - BC^T - I (max-abs of each)."""
    A, B, C, D = blocks(M)
    r1 = np.abs(A @ B.T - B @ A.T).max()
    r2 = np.abs(C @ D.T - D @ C.T).max()
    r3 = np.abs(A @ D.T - B @ C.T - np.eye(2)).max()
    return float(r1), float(r2), float(r3)


def residuals_dual(M):
    """The three residuals of the equivalent form Eq. Intro16:
    A^T C - C^T A, B^T D - D^T B, A^T D - C^T B - I."""
    A, B, C, D = blocks(M)
    r1 = np.abs(A.T @ C - C.T @ A).max()
    r2 = np.abs(B.T @ D - D.T @ B).max()
    r3 = np.abs(A.T @ D - C.T @ B - np.eye(2)).max()
    return float(r1), float(r2), float(r3)


def is_valid(M, tol=TAU_SYM):
    """Eq. Intro12 holds to `tol`."""
    return max(residuals(M)) <= tol


def inverse(M):
    """(A,B;C,D)^{-1} = (D^T, -B^T; -C^T, A^T)  (Eq. CCCMCCCM20)."""
    A, B, C, D = blocks(M)
    return assemble(D.T, -B.T, -C.T, A.T)


def compose(M2, M1):
    """Matrix of the cascade O^{M2} O^{M1} (additivity, Eq. Add12)."""
    return np.asarray(M2, float) @ np.asarray(M1, float)


def J4():
    Z, I = np.zeros((2, 2)), np.eye(2)
    return assemble(Z, I, -I, Z)


def polar_project(M):
    """Nearest-symplectic projection M (M^+ M)^{-1/2}, M^+ = -J M^T J (reading R6).

    The paper prints its matrices to 4 decimals (PAPER.md:1153-1158, 1166-1171,
    1258-1263, 1295-1300), so they violate Eq. Intro12 at ~1e-4; this projects them.
    """
    M = np.asarray(M, float)
    J = J4()
    P = -J @ M.T @ J @ M          # = I exactly when M is symplectic
    w, V = np.linalg.eig(P)
    R = (V @ np.diag(1.0 / np.sqrt(w)) @ np.linalg.inv(V)).real
    return M @ R

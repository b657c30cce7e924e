"""Seeded generators for ABCD matrices and input fields.

Every generator takes a ``numpy.random.Generator`` and returns fp64 (or
complex128) numpy arrays.  Streams: ``config_streams(cfg_id)`` spawns the
(matrix, input) generators from ``SeedSequence(170703688 + cfg_id)``.

Matrices are 4x4 row-major [[A, B], [C, D]] (Eq. Intro04).
The random symplectic generator G(rng) builds M as a product of symplectic
factors (each exactly symplectic by construction); it is a test-input recipe,
not part of the transform.
"""
import math

import numpy as np

__all__ = [
    "SEED_BASE", "config_streams", "rot2", "block", "random_symplectic",
    "dft_matrix4", "idft_matrix4", "gyrator_matrix4", "separable_matrix4",
    "b0_matrix4", "identity4", "iid_cn", "chirp_gauss_field",
    "random_phase_field", "default_dx", "CONFIGS", "c3_sweep_matrices",
]

SEED_BASE = 170703688


def config_streams(cfg_id: int):
    """(matrix_rng, input_rng) for config ``cfg_id`` (SURVEY.md §8(d) 'RNG')."""
    ss = np.random.SeedSequence(SEED_BASE + int(cfg_id))
    a, b = ss.spawn(2)
    return np.random.Generator(np.random.PCG64(a)), np.random.Generator(np.random.PCG64(b))


def default_dx(n: int) -> float:
    """Default spacing sqrt(2*pi/N), so that dx = domega."""
    return math.sqrt(2.0 * math.pi / n)


def rot2(t: float) -> np.ndarray:
    c, s = math.cos(t), math.sin(t)
    return np.array([[c, -s], [s, c]])


def block(A, B, C, D) -> np.ndarray:
    return np.block([[np.asarray(A, float), np.asarray(B, float)],
                     [np.asarray(C, float), np.asarray(D, float)]])


def identity4() -> np.ndarray:
    return np.eye(4)


def dft_matrix4() -> np.ndarray:
    """(0, I; -I, 0): the 2D FT case of Eq. BasicDFT04."""
    I2, Z = np.eye(2), np.zeros((2, 2))
    return block(Z, I2, -I2, Z)


def idft_matrix4() -> np.ndarray:
    """(0, -I; I, 0): the 2D IFT case of Eq. BasicDFT04."""
    I2, Z = np.eye(2), np.zeros((2, 2))
    return block(Z, -I2, I2, Z)


def gyrator_matrix4(alpha: float) -> np.ndarray:
    """Gyrator: (cos a I, sin a J; -sin a J, cos a I), J=[[0,1],[1,0]]."""
    c, s = math.cos(alpha), math.sin(alpha)
    J = np.array([[0.0, 1.0], [1.0, 0.0]])
    return block(c * np.eye(2), s * J, -s * J, c * np.eye(2))


def separable_matrix4(a, b, c) -> np.ndarray:
    """Block-diagonal separable pair of 1D LCTs (a_i, b_i; c_i, d_i), d_i=(1+b_i c_i)/a_i."""
    a = np.asarray(a, float); b = np.asarray(b, float); c = np.asarray(c, float)
    d = (1.0 + b * c) / a
    return block(np.diag(a), np.diag(b), np.diag(c), np.diag(d))


def b0_matrix4(D, S) -> np.ndarray:
    """B = 0 matrix (D^{-T}, 0; S D^{-T}, D), S symmetric (Eq. Intro20)."""
    D = np.asarray(D, float); S = np.asarray(S, float)
    S = 0.5 * (S + S.T)
    Dit = np.linalg.inv(D).T
    return block(Dit, np.zeros((2, 2)), S @ Dit, D)


def random_symplectic(rng: np.random.Generator, min_abs_det_b: float = 0.1,
                      max_tries: int = 1000) -> np.ndarray:
    """G(rng) of SURVEY.md §8(d): M = U (I,0;C,I) (I,S;0,I) diag(Sig, Sig^-1).

    U = diag(R_phi, R_phi) [E F; -F E] diag(R_theta, R_theta) with
    E = diag(cos a, cos b), F = diag(sin a, sin b) (unitary subgroup);
    C, S symmetric with entries ~ U[-2, 2]; Sig = diag(2^u1, 2^u2), u ~ U[-1, 1].
    Redrawn until |det B| > min_abs_det_b.
    """
    for _ in range(max_tries):
        al, be, th, ph = rng.uniform(0.0, 2.0 * math.pi, 4)
        c3 = rng.uniform(-2.0, 2.0, 3)
        s3 = rng.uniform(-2.0, 2.0, 3)
        u = rng.uniform(-1.0, 1.0, 2)
        E = np.diag([math.cos(al), math.cos(be)])
        F = np.diag([math.sin(al), math.sin(be)])
        Rp, Rt = rot2(ph), rot2(th)
        Z = np.zeros((2, 2)); I2 = np.eye(2)
        U = block(Rp, Z, Z, Rp) @ block(E, F, -F, E) @ block(Rt, Z, Z, Rt)
        C = np.array([[c3[0], c3[2]], [c3[2], c3[1]]])
        S = np.array([[s3[0], s3[2]], [s3[2], s3[1]]])
        Sig = np.diag([2.0 ** u[0], 2.0 ** u[1]])
        M = U @ block(I2, Z, C, I2) @ block(I2, S, Z, I2) @ block(Sig, Z, Z, np.linalg.inv(Sig))
        if abs(np.linalg.det(M[0:2, 2:4])) > min_abs_det_b:
            return M
    raise RuntimeError("random_symplectic: no draw with |det B| large enough")


def iid_cn(rng: np.random.Generator, shape) -> np.ndarray:
    """i.i.d. CN(0,1): (N(0,1) + j N(0,1)) / sqrt(2)."""
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    return (re + 1j * im) * (1.0 / math.sqrt(2.0))


def _centered(n: int) -> np.ndarray:
    return np.arange(n) - n // 2


def chirp_gauss_field(rng: np.random.Generator, n: int, batch: int, dx: float = None,
                      noise: float = 0.05) -> np.ndarray:
    """Config-2 input: exp(-|z|^2/(2 sig^2)) exp(j/2 z^T K z) + nu.

    sig = N dx / 8; K symmetric with entries ~ U[-1,1] drawn per image;
    nu ~ noise * rms(clean) * CN(0,1).
    """
    dx = default_dx(n) if dx is None else dx
    x = _centered(n) * dx
    X, Y = np.meshgrid(x, x, indexing="ij")
    sig = n * dx / 8.0
    out = np.empty((batch, n, n), np.complex128)
    env = np.exp(-(X * X + Y * Y) / (2.0 * sig * sig))
    for b in range(batch):
        k = rng.uniform(-1.0, 1.0, 3)
        quad = k[0] * X * X + 2.0 * k[2] * X * Y + k[1] * Y * Y
        clean = env * np.exp(0.5j * quad)
        rms = math.sqrt(float(np.mean(np.abs(clean) ** 2)))
        out[b] = clean + noise * rms * iid_cn(rng, (n, n))
    return out


def random_phase_field(rng: np.random.Generator, shape) -> np.ndarray:
    """Config-3 input: unit amplitude, phase 2*pi*U[0,1)."""
    return np.exp(2j * math.pi * rng.uniform(0.0, 1.0, shape))


def c3_sweep_matrices(rng: np.random.Generator) -> dict:
    """Config-3 special-case sweep (BASELINE.json configs[2]), drawn in
    this order from the config's matrix stream: the 2D DFT (0,I;-I,0); a gyrator with
    alpha ~ U[0,pi), redrawn while sin^2 alpha <= 0.1; a separable pair with a_i, b_i, c_i
    ~ U[-2,2], |b_i| > 0.32, |a_i| > 0.1; and a B = 0 matrix (D^-T, 0; S D^-T, D) with
    D ~ U[-2,2], 0.5 <= |det D| <= 2, S ~ U[-2,2] symmetrised."""
    subs = {"dft": dft_matrix4()}
    while True:
        a = rng.uniform(0, math.pi)
        if math.sin(a) ** 2 > 0.1:
            break
    subs["gyrator"] = gyrator_matrix4(a)
    while True:
        a = rng.uniform(-2, 2, 2)
        b = rng.uniform(-2, 2, 2)
        c = rng.uniform(-2, 2, 2)
        if np.all(np.abs(b) > 0.32) and np.all(np.abs(a) > 0.1):
            break
    subs["separable"] = separable_matrix4(a, b, c)
    while True:
        D = rng.uniform(-2, 2, (2, 2))
        if 0.5 <= abs(np.linalg.det(D)) <= 2:
            break
    S = rng.uniform(-2, 2, (2, 2))
    subs["b0"] = b0_matrix4(D, S)
    return subs


CONFIGS = {
    1: dict(n=32, dtype="c128", batch=1, kind="random"),
    2: dict(n=256, dtype="c64", batch=64, kind="random"),
    3: dict(n=1024, dtype="c64", batch=16, kind="sweep"),
    4: dict(n=4096, dtype="c64", batch=32, kind="random"),
    5: dict(n=16384, dtype="c64", batch=1, kind="random"),
}

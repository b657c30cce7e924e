"""Decomposition planner (oracle; test infrastructure only, see oracle/__init__.py).

Follows PAPER.md §4 in the paper's notation:

* CM-CC-CM-CC (form I), Eq. Bnonsym04-12:
      (A,B;C,D) = CM((D'-I)B'^{-1}) CC(B') CM(B'^{-1}(A-I)) CC(H),
      B' = B - A H,  D' = D - C H,  H = H^T,  B' = B'^T,  det B' != 0.
* Feasible set: B' symmetric  <=>  v . h = rhs with
      h = (h11, h22, h12), v = (a21, -a12, a22 - a11), rhs = b21 - b12
  (the 1,2 and 2,1 entries of B - A H equated).
* HA objective, Eq. HA16/HA24:
      J(H) = gamma((D'-I)B'^{-1}) gamma(B') gamma(B'^{-1}(A-I)) gamma(H),
      gamma(C) = (|c11| + |c12| + 1)(|c12| + |c22| + 1).
  The paper gives no search procedure; reading R5 fixes one
  (multi-scale grid + Nelder-Mead + deterministic ties), implemented here.
* LC rule, Eq. LC08/LC10: H = (h,0;0,0), h = (b21-b12)/a21,
  or H = (0,0;0,h), h = (b12-b21)/a12; pick the lower J; fall back to HA when
  neither applies or det B' = 0.
* CC-CM-CC-CM (form II), Eq. CCCMCCCM08-16 with
  H1 = -H~ where H~ is the form-I choice for M^{-1}.
* Reversible dispatch, Eq. Reversible08: form I when
  tr B > 0, form II when tr B < 0; reading R7 extends the key to
  tr B = 0 by an odd lexicographic key.

A plan is a dict; `chain` is the list of operators in application order
(first applied first) as tuples ('CM', Q) on the space grid or ('CC', B).
"""
import math

import numpy as np

from .symplectic import blocks, is_valid, inverse, residuals

DET_REL = 1e-8        # |det B'| > DET_REL * max(1, |B'|_max^2)   (reading R5)
KEY_TOL = 1e-12       # dispatch-key zero threshold (reading R7)
TIE_REL = 1e-12       # relative objective tie (reading R5)
SCALES = (0.25, 1.0, 4.0, 16.0)   # plus R = 4 (1 + |M|_max)  (reading R5)
GRID_PTS = 21
NM_STARTS = 12
NM_XATOL = 1e-10
NM_MAXIT = 4000


class PlanError(Exception):
    pass


def sym(X):
    return 0.5 * (X + X.T)


def gamma(Cm):
    """Ratio function gamma(C) of Eq. HA16, C symmetric."""
    c11, c22 = Cm[0, 0], Cm[1, 1]
    c12 = 0.5 * (Cm[0, 1] + Cm[1, 0])
    return (abs(c11) + abs(c12) + 1.0) * (abs(c12) + abs(c22) + 1.0)


def hmat(h):
    """h = (h11, h22, h12) -> symmetric H."""
    return np.array([[h[0], h[2]], [h[2], h[1]]], dtype=np.float64)


def _inv2(X):
    """Inverse of a 2x2 matrix by the adjugate formula."""
    det = X[0, 0] * X[1, 1] - X[0, 1] * X[1, 0]
    return np.array([[X[1, 1], -X[0, 1]], [-X[1, 0], X[0, 0]]]) / det


def form1_stages(M, H):
    """B', D', P2 = B'^{-1}(A-I), P4 = (D'-I)B'^{-1} for a given symmetric H
    (Eq. Bnonsym04-08).  Returns None if B' is singular
    in the sense of reading R5."""
    A, B, C, D = blocks(M)
    I = np.eye(2)
    Bp = B - A @ H
    Dp = D - C @ H
    det = Bp[0, 0] * Bp[1, 1] - Bp[0, 1] * Bp[1, 0]
    if not abs(det) > DET_REL * max(1.0, np.abs(Bp).max() ** 2):
        return None
    Bpi = _inv2(Bp)
    P2 = Bpi @ (A - I)
    P4 = (Dp - I) @ Bpi
    return dict(H=sym(H), Bp=sym(Bp), Dp=Dp, P2=sym(P2), P4=sym(P4))


def objective(M, H):
    """J(H) of Eq. HA24; +inf when infeasible (det B' = 0)."""
    st = form1_stages(M, H)
    if st is None:
        return math.inf
    return gamma(st["P4"]) * gamma(st["Bp"]) * gamma(st["P2"]) * gamma(st["H"])


def objective_many(M, hs):
    """objective() for many h = (h11, h22, h12) rows at once (same formulas, vectorised)."""
    A, B, C, D = blocks(M)
    hs = np.asarray(hs, float)
    H = np.empty((hs.shape[0], 2, 2))
    H[:, 0, 0], H[:, 1, 1], H[:, 0, 1], H[:, 1, 0] = hs[:, 0], hs[:, 1], hs[:, 2], hs[:, 2]
    I = np.eye(2)
    Bp = B[None] - A[None] @ H
    Dp = D[None] - C[None] @ H
    det = Bp[:, 0, 0] * Bp[:, 1, 1] - Bp[:, 0, 1] * Bp[:, 1, 0]
    ok = np.abs(det) > DET_REL * np.maximum(1.0, np.abs(Bp).max(axis=(1, 2)) ** 2)
    adj = np.empty_like(Bp)
    adj[:, 0, 0], adj[:, 0, 1] = Bp[:, 1, 1], -Bp[:, 0, 1]
    adj[:, 1, 0], adj[:, 1, 1] = -Bp[:, 1, 0], Bp[:, 0, 0]
    with np.errstate(divide="ignore", invalid="ignore"):
        Bpi = adj / det[:, None, None]
        P2 = Bpi @ (A - I)[None]
        P4 = (Dp - I[None]) @ Bpi

    def g(X):
        c12 = 0.5 * (X[:, 0, 1] + X[:, 1, 0])
        return (np.abs(X[:, 0, 0]) + np.abs(c12) + 1.0) * (np.abs(c12) + np.abs(X[:, 1, 1]) + 1.0)

    with np.errstate(invalid="ignore", over="ignore"):
        J = g(P4) * g(Bp) * g(P2) * g(H)
    return np.where(ok & np.isfinite(J), J, math.inf)


def feasible_param(M):
    """Affine parametrisation h = h0 + Nb t of {H = H^T : B - AH symmetric}
    (reading R5).  Returns (h0, Nb) with Nb of shape (3, k)."""
    A, B, C, D = blocks(M)
    v = np.array([A[1, 0], -A[0, 1], A[1, 1] - A[0, 0]])
    rhs = B[1, 0] - B[0, 1]
    nA = np.abs(A).max()
    vn = float(np.linalg.norm(v))
    if vn <= 1e-12 * nA or vn == 0.0:
        # A = a I: every symmetric H keeps B' = B - aH symmetric iff B is.
        if abs(rhs) > 1e-10 * max(1.0, np.abs(B).max()):
            raise PlanError("NO_DECOMP: A = aI with B nonsymmetric (reading R5, PAPER.md:681)")
        return np.zeros(3), np.eye(3)
    h0 = v * (rhs / (vn * vn))
    vh = v / vn
    a = int(np.argmin(np.abs(vh)))          # first index of smallest |v_i|
    e = np.zeros(3)
    e[a] = 1.0
    u1 = e - vh[a] * vh
    u1 /= np.linalg.norm(u1)
    u2 = np.cross(vh, u1)
    return h0, np.stack([u1, u2], axis=1)


def _key(J, h):
    """Ordering for candidates: objective, then |H|_F, then (h11, h22, h12)."""
    return (J, h[0] ** 2 + h[1] ** 2 + 2 * h[2] ** 2, h[0], h[1], h[2])


def _better(J1, h1, J2, h2):
    """True when candidate 1 is strictly preferred to candidate 2 (reading R5)."""
    if J2 == math.inf:
        return J1 < math.inf
    if J1 < J2 * (1.0 - TIE_REL):
        return True
    if J2 < J1 * (1.0 - TIE_REL):
        return False
    n1 = h1[0] ** 2 + h1[1] ** 2 + 2 * h1[2] ** 2
    n2 = h2[0] ** 2 + h2[1] ** 2 + 2 * h2[2] ** 2
    if n1 != n2:
        return n1 < n2
    return tuple(h1) < tuple(h2)


def nelder_mead(f, x0, step):
    """Plain Nelder-Mead (reflection 1, expansion 2, contraction 1/2, shrink 1/2),
    stopping when the simplex diameter < NM_XATOL (reading R5)."""
    k = len(x0)
    simplex = [np.array(x0, float)]
    for i in range(k):
        x = np.array(x0, float)
        x[i] += step
        simplex.append(x)
    fv = [f(x) for x in simplex]
    for _ in range(NM_MAXIT):
        order = sorted(range(k + 1), key=lambda i: (fv[i], i))
        simplex = [simplex[i] for i in order]
        fv = [fv[i] for i in order]
        diam = max(float(np.abs(simplex[i] - simplex[0]).max()) for i in range(1, k + 1))
        if diam < NM_XATOL:
            break
        cen = sum(simplex[:k]) / k
        xr = cen + (cen - simplex[k])
        fr = f(xr)
        if fr < fv[0]:
            xe = cen + 2.0 * (cen - simplex[k])
            fe = f(xe)
            if fe < fr:
                simplex[k], fv[k] = xe, fe
            else:
                simplex[k], fv[k] = xr, fr
        elif fr < fv[k - 1]:
            simplex[k], fv[k] = xr, fr
        else:
            if fr < fv[k]:
                xc = cen + 0.5 * (xr - cen)      # outside contraction
            else:
                xc = cen + 0.5 * (simplex[k] - cen)  # inside contraction
            fc = f(xc)
            if fc < min(fr, fv[k]):
                simplex[k], fv[k] = xc, fc
            else:
                for i in range(1, k + 1):
                    simplex[i] = simplex[0] + 0.5 * (simplex[i] - simplex[0])
                    fv[i] = f(simplex[i])
    i0 = min(range(k + 1), key=lambda i: (fv[i], i))
    return simplex[i0], fv[i0]


def ha_search(M):
    """HA choice of H (Eq. HA24) by the search of reading R5.
    Returns (h, J) with h = (h11, h22, h12)."""
    h0, Nb = feasible_param(M)
    k = Nb.shape[1]
    R = 4.0 * (1.0 + float(np.abs(M).max()))

    def f(t):
        return objective(M, hmat(h0 + Nb @ np.asarray(t, float)))

    ts = []
    for s in SCALES + (R,):
        g = np.linspace(-s, s, GRID_PTS)
        mesh = np.meshgrid(*([g] * k), indexing="ij")
        ts.append(np.stack([m.ravel() for m in mesh], axis=1))
    # H = 0 and the two LC candidates, when they lie on the feasible plane.
    specials = [np.zeros(3)]
    A, B, _, _ = blocks(M)
    if A[1, 0] != 0.0:
        specials.append(np.array([(B[1, 0] - B[0, 1]) / A[1, 0], 0.0, 0.0]))
    if A[0, 1] != 0.0:
        specials.append(np.array([0.0, (B[0, 1] - B[1, 0]) / A[0, 1], 0.0]))
    for hs in specials:
        t = Nb.T @ (hs - h0)
        if np.abs(h0 + Nb @ t - hs).max() <= 1e-12 * max(1.0, np.abs(hs).max()):
            ts.append(t[None, :])
    ts = np.unique(np.concatenate(ts), axis=0)
    hs = h0[None, :] + ts @ Nb.T
    Js = objective_many(M, hs)
    ok = np.isfinite(Js)
    if not ok.any():
        raise PlanError("NO_DECOMP: no feasible H found (reading R5)")
    ts, hs, Js = ts[ok], hs[ok], Js[ok]
    norm = hs[:, 0] ** 2 + hs[:, 1] ** 2 + 2 * hs[:, 2] ** 2
    order = np.lexsort((hs[:, 2], hs[:, 1], hs[:, 0], norm, Js))   # = _key order
    best_h, best_J = hs[order[0]], float(Js[order[0]])
    items = [(float(Js[i]), ts[i]) for i in order[:NM_STARTS]]
    for J0, t0 in items[:NM_STARTS]:
        step = 0.05 * max(1.0, float(np.abs(t0).max()))
        t, J = nelder_mead(f, t0, step)
        h = h0 + Nb @ t
        if _better(J, h, best_J, best_h):
            best_h, best_J = h, J
    return np.asarray(best_h, float), float(best_J)


def lc_choice(M):
    """LC choice of H (Eq. LC04-10).  Returns (h-vector, J, axis)
    where axis = 'x' for H = (h,0;0,0), 'y' for H = (0,0;0,h); None if neither
    form applies or both give singular B' (then the caller falls back to HA)."""
    A, B, _, _ = blocks(M)
    best = None
    if A[1, 0] != 0.0:
        h = np.array([(B[1, 0] - B[0, 1]) / A[1, 0], 0.0, 0.0])
        J = objective(M, hmat(h))
        if J < math.inf:
            best = (h, J, "x")
    if A[0, 1] != 0.0:
        h = np.array([0.0, (B[0, 1] - B[1, 0]) / A[0, 1], 0.0])
        J = objective(M, hmat(h))
        if J < math.inf and (best is None or J < best[1]):
            best = (h, J, "y")
    return best


def dispatch_key(M):
    """Odd dispatch key s(M) (reading R7 extending Eq. Reversible08):
    the first of (tr B, b12+b21, b11, tr A - tr D, a12+a21-d12-d21) that is nonzero.
    Every entry changes sign under M -> M^{-1} = (D^T, -B^T; -C^T, A^T)."""
    A, B, C, D = blocks(M)
    tol = KEY_TOL * max(1.0, float(np.abs(M).max()))
    for s in (np.trace(B), B[0, 1] + B[1, 0], B[0, 0], np.trace(A) - np.trace(D),
              A[0, 1] + A[1, 0] - D[0, 1] - D[1, 0]):
        if abs(s) > tol:
            return float(s)
    return 0.0


def is_b_zero(M):
    """B = 0 case of Eq. Intro20 (reading R10): |B|_max <= 1e-12 max(1, |M|_max)."""
    _, B, _, _ = blocks(M)
    return float(np.abs(B).max()) <= 1e-12 * max(1.0, float(np.abs(M).max()))


def choose_h(M, variant="HA"):
    """H for the form-I decomposition of M (HA search or LC rule with HA fallback)."""
    if variant == "LC":
        lc = lc_choice(M)
        if lc is not None:
            return lc[0], lc[1], lc[2]
    h, J = ha_search(M)
    return h, J, None


def plan(M, variant="HA", policy="reversible", h_override=None):
    """Full plan of the NsDLCT for M.

    policy: 'reversible' = Eq. Reversible08 + reading R7 (default);
            'formI' = CM-CC-CM-CC always (reading R8, used for the paper's §5 numbers).
    h_override: use this H (form I) / H~ (form II, the form-I H of M^{-1})
                instead of searching (used to align with a given plan).
    """
    M = np.asarray(M, float)
    if not is_valid(M):
        raise PlanError("NOT_SYMPLECTIC: Eq. Intro12 residual %.3g" % max(residuals(M)))
    if is_b_zero(M):
        A, B, C, D = blocks(M)
        return dict(kind="B0", M=M, C=C, D=D, chain=[("B0", C, D)])
    key = dispatch_key(M)
    form = "I" if (policy == "formI" or key >= 0.0) else "II"
    if form == "I":
        if h_override is not None:
            h, J, axis = np.asarray(h_override, float), objective(M, hmat(h_override)), None
        else:
            h, J, axis = choose_h(M, variant)
        H = hmat(h)
        st = form1_stages(M, H)
        if st is None:
            raise PlanError("NO_DECOMP: det B' = 0 for the chosen H")
        # Eq. HA28: CM(P4) CC(B') CM(P2) CC(H), applied right to left.
        chain = [("CC", st["H"]), ("CM", st["P2"]), ("CC", st["Bp"]), ("CM", st["P4"])]
        return dict(kind="I", M=M, h=h, J=J, axis=axis, H=st["H"], Bp=st["Bp"],
                    P2=st["P2"], P4=st["P4"], chain=chain, key=key)
    # Form II (Eq. CCCMCCCM08-16) with H1 = -H~, H~ the form-I
    # choice for M~ = M^{-1}.
    Mt = inverse(M)
    if h_override is not None:
        ht, J, axis = np.asarray(h_override, float), objective(Mt, hmat(h_override)), None
    else:
        ht, J, axis = choose_h(Mt, variant)
    H1 = -hmat(ht)
    A1, B1, C1, D1 = blocks(M)
    I = np.eye(2)
    B1p = B1 - H1 @ D1            # Eq. CCCMCCCM08
    A1p = A1 - H1 @ C1
    det = B1p[0, 0] * B1p[1, 1] - B1p[0, 1] * B1p[1, 0]
    if not abs(det) > DET_REL * max(1.0, np.abs(B1p).max() ** 2):
        raise PlanError("NO_DECOMP: det B1' = 0")
    B1pi = np.linalg.inv(B1p)
    Q_left = sym((D1 - I) @ B1pi)     # CM((D1 - I) B1'^{-1})
    Q_right = sym(B1pi @ (A1p - I))   # CM(B1'^{-1}(A1' - I))
    # Eq. CCCMCCCM16: CC(H1) CM(Q_left) CC(B1') CM(Q_right).
    chain = [("CM", Q_right), ("CC", sym(B1p)), ("CM", Q_left), ("CC", sym(H1))]
    return dict(kind="II", M=M, h=ht, J=J, axis=axis, H1=sym(H1), B1p=sym(B1p),
                Q_left=Q_left, Q_right=Q_right, chain=chain, key=key)


def chain_matrix(chain):
    """4x4 matrix of a CM/CC chain (CM(Q) = (I,0;Q,I), CC(B) = (I,B;0,I),
    Eq. BasicCM04 / BasicCC04), for the recomposition check."""
    I, Z = np.eye(2), np.zeros((2, 2))
    T = np.eye(4)
    for op in chain:
        if op[0] == "CM":
            F = np.block([[I, Z], [op[1], I]])
        elif op[0] == "CC":
            F = np.block([[I, op[1]], [Z, I]])
        else:
            raise ValueError(op[0])
        T = F @ T
    return T

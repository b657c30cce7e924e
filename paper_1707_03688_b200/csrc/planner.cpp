// Host-side planner of the 2D NsDLCT (arxiv 1707.03688), C++17, no CUDA.
//
// Given the ABCD matrix M (Eq. Intro04) this decides, entirely on the
// host and in fp64, which chain of chirp multiplications (CM) and chirp convolutions
// (CC) the device executes:
//   * validity, Eq. Intro12, tolerance 1e-10 (reading R6);
//   * B = 0 -> Eq. Intro20, chirp x affine (reading R10);
//   * dispatch key s(M) (Eq. Reversible08, extended by reading R7);
//   * form I (CM-CC-CM-CC, Eq. Bnonsym08/HA28) for s >= 0,
//     otherwise form II as the exact inverse of form I of M^-1 (Eq. CCCMCCCM30,
//     PAPER.md:999-1006):  O_II(M) = CC(-H~) CM(-P2~) CC(-B'~) CM(-P4~);
//   * H by the HA objective of Eq. HA24 with the deterministic search
//     of reading R5, or the LC rule of Eq. LC08/LC10.
// The executed chain is stored as five symmetric chirp matrices Q0..Q4:
//   G = CM_r(Q4) F^-1 CM_w(Q3) F CM_r(Q2) F^-1 CM_w(Q1) F CM_r(Q0) g
// (CC(B) = F^-1 CM_w(-B) F, Eq. BasicCC20).
#include "planner.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <limits>
#include <vector>

namespace nslct {
namespace {

constexpr double kTauSym = 1e-10;
constexpr double kDetRel = 1e-8;
constexpr double kKeyTol = 1e-12;
constexpr double kTieRel = 1e-12;
constexpr int kGridPts = 21;
constexpr int kNmStarts = 12;
constexpr double kNmXatol = 1e-10;
constexpr int kNmMaxit = 4000;
constexpr double kInf = std::numeric_limits<double>::infinity();

M2 mul(const M2& x, const M2& y) {
  return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c,
          x.c * y.b + x.d * y.d};
}
M2 sub(const M2& x, const M2& y) { return {x.a - y.a, x.b - y.b, x.c - y.c, x.d - y.d}; }
M2 add(const M2& x, const M2& y) { return {x.a + y.a, x.b + y.b, x.c + y.c, x.d + y.d}; }
M2 tr(const M2& x) { return {x.a, x.c, x.b, x.d}; }
M2 neg(const M2& x) { return {-x.a, -x.b, -x.c, -x.d}; }
M2 eye() { return {1, 0, 0, 1}; }
double det(const M2& x) { return x.a * x.d - x.b * x.c; }
double maxabs(const M2& x) {
  return std::max(std::max(std::fabs(x.a), std::fabs(x.b)), std::max(std::fabs(x.c), std::fabs(x.d)));
}
M2 inv(const M2& x) {  // adjugate / det
  double dt = det(x);
  return {x.d / dt, -x.b / dt, -x.c / dt, x.a / dt};
}
M2 of(const Sym& s) { return {s.q11, s.q12, s.q12, s.q22}; }
Sym symm(const M2& x) { return {x.a, x.d, 0.5 * (x.b + x.c)}; }
Sym negs(const Sym& s) { return {-s.q11, -s.q22, -s.q12}; }

struct Blocks {
  M2 A, B, C, D;
};
Blocks blocks(const double m[16]) {
  return {{m[0], m[1], m[4], m[5]}, {m[2], m[3], m[6], m[7]},
          {m[8], m[9], m[12], m[13]}, {m[10], m[11], m[14], m[15]}};
}
void unblocks(const Blocks& b, double m[16]) {
  const M2* bl[4] = {&b.A, &b.B, &b.C, &b.D};
  for (int k = 0; k < 4; ++k) {
    int r0 = (k / 2) * 2, c0 = (k % 2) * 2;
    m[r0 * 4 + c0] = bl[k]->a;
    m[r0 * 4 + c0 + 1] = bl[k]->b;
    m[(r0 + 1) * 4 + c0] = bl[k]->c;
    m[(r0 + 1) * 4 + c0 + 1] = bl[k]->d;
  }
}

// (A,B;C,D)^-1 = (D^T, -B^T; -C^T, A^T)  (Eq. CCCMCCCM20)
void inverse4(const double m[16], double out[16]) {
  Blocks b = blocks(m);
  Blocks r{tr(b.D), neg(tr(b.B)), neg(tr(b.C)), tr(b.A)};
  unblocks(r, out);
}

double sym_residual(const double m[16]) {  // Eq. Intro12
  Blocks b = blocks(m);
  double r1 = maxabs(sub(mul(b.A, tr(b.B)), mul(b.B, tr(b.A))));
  double r2 = maxabs(sub(mul(b.C, tr(b.D)), mul(b.D, tr(b.C))));
  double r3 = maxabs(sub(sub(mul(b.A, tr(b.D)), mul(b.B, tr(b.C))), eye()));
  return std::max(r1, std::max(r2, r3));
}

double maxabs16(const double m[16]) {
  double r = 0;
  for (int i = 0; i < 16; ++i) r = std::max(r, std::fabs(m[i]));
  return r;
}

struct Stages {
  bool ok;
  Sym H, Bp, P2, P4;
};

// B' = B - AH, D' = D - CH, P2 = B'^-1 (A - I), P4 = (D' - I) B'^-1  (Eq. Bnonsym04-08)
Stages form1(const Blocks& b, const Sym& Hs) {
  Stages s{};
  M2 H = of(Hs);
  M2 Bp = sub(b.B, mul(b.A, H));
  M2 Dp = sub(b.D, mul(b.C, H));
  double dt = Bp.a * Bp.d - Bp.b * Bp.c;
  double nb = maxabs(Bp);
  if (!(std::fabs(dt) > kDetRel * std::max(1.0, nb * nb))) {
    s.ok = false;
    return s;
  }
  M2 Bpi = inv(Bp);
  M2 P2 = mul(Bpi, sub(b.A, eye()));
  M2 P4 = mul(sub(Dp, eye()), Bpi);
  s.ok = true;
  s.H = Hs;
  s.Bp = symm(Bp);
  s.P2 = symm(P2);
  s.P4 = symm(P4);
  return s;
}

double objective_b(const Blocks& b, const Sym& H) {
  Stages s = form1(b, H);
  if (!s.ok) return kInf;
  double J = gamma_ratio(s.P4) * gamma_ratio(s.Bp) * gamma_ratio(s.P2) * gamma_ratio(s.H);
  return std::isfinite(J) ? J : kInf;
}

using V3 = std::array<double, 3>;

Sym hsym(const V3& h) { return {h[0], h[1], h[2]}; }

double hnorm(const V3& h) { return h[0] * h[0] + h[1] * h[1] + 2 * h[2] * h[2]; }

bool better(double J1, const V3& h1, double J2, const V3& h2) {
  if (J2 == kInf) return J1 < kInf;
  if (J1 < J2 * (1.0 - kTieRel)) return true;
  if (J2 < J1 * (1.0 - kTieRel)) return false;
  double n1 = hnorm(h1), n2 = hnorm(h2);
  if (n1 != n2) return n1 < n2;
  return h1 < h2;
}

struct Param {
  int k;           // 2 or 3
  V3 h0;
  double Nb[3][3]; // columns = basis vectors (first k used)
};

V3 h_of(const Param& P, const double* t) {
  V3 h = P.h0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < P.k; ++j) h[i] += P.Nb[i][j] * t[j];
  return h;
}

// Feasible plane {H = H^T : B - AH symmetric}:
// v . h = rhs, h = (h11, h22, h12), v = (a21, -a12, a22 - a11), rhs = b21 - b12.
int feasible(const Blocks& b, Param* P, std::string* err) {
  double v[3] = {b.A.c, -b.A.b, b.A.d - b.A.a};
  double rhs = b.B.c - b.B.b;
  double nA = maxabs(b.A);
  double vn = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  if (vn <= 1e-12 * nA || vn == 0.0) {
    if (std::fabs(rhs) > 1e-10 * std::max(1.0, maxabs(b.B))) {
      *err = "A = aI with B nonsymmetric: no CM-CC-CM-CC decomposition (reading R5)";
      return 3;
    }
    P->k = 3;
    P->h0 = {0, 0, 0};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) P->Nb[i][j] = (i == j) ? 1.0 : 0.0;
    return 0;
  }
  P->k = 2;
  double s = rhs / (vn * vn);
  P->h0 = {v[0] * s, v[1] * s, v[2] * s};
  double vh[3] = {v[0] / vn, v[1] / vn, v[2] / vn};
  int a = 0;
  for (int i = 1; i < 3; ++i)
    if (std::fabs(vh[i]) < std::fabs(vh[a])) a = i;
  double u1[3];
  for (int i = 0; i < 3; ++i) u1[i] = (i == a ? 1.0 : 0.0) - vh[a] * vh[i];
  double un = std::sqrt(u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2]);
  for (int i = 0; i < 3; ++i) u1[i] /= un;
  double u2[3] = {vh[1] * u1[2] - vh[2] * u1[1], vh[2] * u1[0] - vh[0] * u1[2],
                  vh[0] * u1[1] - vh[1] * u1[0]};
  for (int i = 0; i < 3; ++i) {
    P->Nb[i][0] = u1[i];
    P->Nb[i][1] = u2[i];
    P->Nb[i][2] = 0.0;
  }
  return 0;
}

// Plain Nelder-Mead (reflection 1, expansion 2, contraction 1/2, shrink 1/2), reading R5.
template <class F>
double nelder_mead(F&& f, int k, double* x0, double step) {
  std::vector<std::array<double, 3>> sx(k + 1);
  std::vector<double> fv(k + 1);
  for (int i = 0; i <= k; ++i) {
    for (int j = 0; j < 3; ++j) sx[i][j] = (j < k) ? x0[j] : 0.0;
    if (i > 0) sx[i][i - 1] += step;
    fv[i] = f(sx[i].data());
  }
  std::vector<int> ord(k + 1);
  for (int it = 0; it < kNmMaxit; ++it) {
    for (int i = 0; i <= k; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return fv[a] < fv[b]; });
    auto sx2 = sx;
    auto fv2 = fv;
    for (int i = 0; i <= k; ++i) {
      sx[i] = sx2[ord[i]];
      fv[i] = fv2[ord[i]];
    }
    double diam = 0;
    for (int i = 1; i <= k; ++i)
      for (int j = 0; j < k; ++j) diam = std::max(diam, std::fabs(sx[i][j] - sx[0][j]));
    if (diam < kNmXatol) break;
    std::array<double, 3> cen{0, 0, 0}, xr{}, xe{}, xc{};
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) cen[j] += sx[i][j];
    for (int j = 0; j < k; ++j) cen[j] /= k;
    for (int j = 0; j < k; ++j) xr[j] = cen[j] + (cen[j] - sx[k][j]);
    double fr = f(xr.data());
    if (fr < fv[0]) {
      for (int j = 0; j < k; ++j) xe[j] = cen[j] + 2.0 * (cen[j] - sx[k][j]);
      double fe = f(xe.data());
      if (fe < fr) {
        sx[k] = xe;
        fv[k] = fe;
      } else {
        sx[k] = xr;
        fv[k] = fr;
      }
    } else if (fr < fv[k - 1]) {
      sx[k] = xr;
      fv[k] = fr;
    } else {
      if (fr < fv[k])
        for (int j = 0; j < k; ++j) xc[j] = cen[j] + 0.5 * (xr[j] - cen[j]);
      else
        for (int j = 0; j < k; ++j) xc[j] = cen[j] + 0.5 * (sx[k][j] - cen[j]);
      double fc = f(xc.data());
      if (fc < std::min(fr, fv[k])) {
        sx[k] = xc;
        fv[k] = fc;
      } else {
        for (int i = 1; i <= k; ++i) {
          for (int j = 0; j < k; ++j) sx[i][j] = sx[0][j] + 0.5 * (sx[i][j] - sx[0][j]);
          fv[i] = f(sx[i].data());
        }
      }
    }
  }
  int i0 = 0;
  for (int i = 1; i <= k; ++i)
    if (fv[i] < fv[i0]) i0 = i;
  for (int j = 0; j < k; ++j) x0[j] = sx[i0][j];
  return fv[i0];
}

int search(const Blocks& b, double mmax, V3* hbest, double* Jbest, std::string* err) {
  Param P;
  int st = feasible(b, &P, err);
  if (st) return st;
  const int k = P.k;
  const double R = 4.0 * (1.0 + mmax);
  const double scales[5] = {0.25, 1.0, 4.0, 16.0, R};
  std::vector<std::array<double, 3>> ts;
  for (double s : scales) {
    double g[kGridPts];
    double step = (s - (-s)) / (kGridPts - 1);  // numpy.linspace arithmetic
    for (int i = 0; i < kGridPts; ++i) g[i] = -s + i * step;
    g[kGridPts - 1] = s;
    if (k == 2) {
      for (int i = 0; i < kGridPts; ++i)
        for (int j = 0; j < kGridPts; ++j) ts.push_back({g[i], g[j], 0.0});
    } else {
      for (int i = 0; i < kGridPts; ++i)
        for (int j = 0; j < kGridPts; ++j)
          for (int l = 0; l < kGridPts; ++l) ts.push_back({g[i], g[j], g[l]});
    }
  }
  // H = 0 and the LC candidates (Eq. LC08/LC10) when on the feasible plane
  std::vector<V3> specials;
  specials.push_back({0, 0, 0});
  if (b.A.c != 0.0) specials.push_back({(b.B.c - b.B.b) / b.A.c, 0.0, 0.0});
  if (b.A.b != 0.0) specials.push_back({0.0, (b.B.b - b.B.c) / b.A.b, 0.0});
  for (const V3& hs : specials) {
    double t[3] = {0, 0, 0};
    for (int j = 0; j < k; ++j)
      for (int i = 0; i < 3; ++i) t[j] += P.Nb[i][j] * (hs[i] - P.h0[i]);
    V3 hb = h_of(P, t);
    double dev = 0, hm = 0;
    for (int i = 0; i < 3; ++i) {
      dev = std::max(dev, std::fabs(hb[i] - hs[i]));
      hm = std::max(hm, std::fabs(hs[i]));
    }
    if (dev <= 1e-12 * std::max(1.0, hm)) ts.push_back({t[0], t[1], t[2]});
  }
  std::sort(ts.begin(), ts.end());
  ts.erase(std::unique(ts.begin(), ts.end()), ts.end());

  struct Cand {
    double J, nrm;
    V3 h;
    std::array<double, 3> t;
  };
  std::vector<Cand> cs;
  cs.reserve(ts.size());
  for (auto& t : ts) {
    V3 h = h_of(P, t.data());
    double J = objective_b(b, hsym(h));
    if (J < kInf) cs.push_back({J, hnorm(h), h, t});
  }
  if (cs.empty()) {
    *err = "no feasible H found (reading R5)";
    return 3;
  }
  std::sort(cs.begin(), cs.end(), [](const Cand& x, const Cand& y) {
    if (x.J != y.J) return x.J < y.J;
    if (x.nrm != y.nrm) return x.nrm < y.nrm;
    return x.h < y.h;
  });
  V3 bh = cs[0].h;
  double bJ = cs[0].J;
  auto f = [&](const double* t) { return objective_b(b, hsym(h_of(P, t))); };
  int nst = std::min<int>(kNmStarts, (int)cs.size());
  for (int s = 0; s < nst; ++s) {
    double t[3] = {cs[s].t[0], cs[s].t[1], cs[s].t[2]};
    double tm = 0;
    for (int j = 0; j < k; ++j) tm = std::max(tm, std::fabs(t[j]));
    double J = nelder_mead(f, k, t, 0.05 * std::max(1.0, tm));
    V3 h = h_of(P, t);
    if (better(J, h, bJ, bh)) {
      bh = h;
      bJ = J;
    }
  }
  *hbest = bh;
  *Jbest = bJ;
  return 0;
}

// LC rule (Eq. LC08/LC10): candidates (h,0;0,0) and (0,0;0,h); pick lower J.
bool lc_choice(const Blocks& b, V3* h, double* J, int* axis) {
  bool found = false;
  if (b.A.c != 0.0) {
    V3 hx = {(b.B.c - b.B.b) / b.A.c, 0.0, 0.0};
    double Jx = objective_b(b, hsym(hx));
    if (Jx < kInf) {
      *h = hx;
      *J = Jx;
      *axis = 1;
      found = true;
    }
  }
  if (b.A.b != 0.0) {
    V3 hy = {0.0, (b.B.b - b.B.c) / b.A.b, 0.0};
    double Jy = objective_b(b, hsym(hy));
    if (Jy < kInf && (!found || Jy < *J)) {
      *h = hy;
      *J = Jy;
      *axis = 2;
      found = true;
    }
  }
  return found;
}

double dispatch_key(const double m[16]) {  // reading R7
  Blocks b = blocks(m);
  double tol = kKeyTol * std::max(1.0, maxabs16(m));
  double keys[5] = {b.B.a + b.B.d, b.B.b + b.B.c, b.B.a, (b.A.a + b.A.d) - (b.D.a + b.D.d),
                    b.A.b + b.A.c - b.D.b - b.D.c};
  for (double s : keys)
    if (std::fabs(s) > tol) return s;
  return 0.0;
}

// 4x4 product of the executed chain, M = CM(Q4) CC(-Q3) CM(Q2) CC(-Q1) CM(Q0)
void chain_matrix(const Plan& p, double out[16]) {
  double T[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
  auto apply = [&](bool cm, const Sym& q) {
    double F[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
    int r0 = cm ? 2 : 0, c0 = cm ? 0 : 2;
    double s = cm ? 1.0 : -1.0;
    F[r0 * 4 + c0] = s * q.q11;
    F[r0 * 4 + c0 + 1] = s * q.q12;
    F[(r0 + 1) * 4 + c0] = s * q.q12;
    F[(r0 + 1) * 4 + c0 + 1] = s * q.q22;
    double R[16];
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        double acc = 0;
        for (int l = 0; l < 4; ++l) acc += F[i * 4 + l] * T[l * 4 + j];
        R[i * 4 + j] = acc;
      }
    std::copy(R, R + 16, T);
  };
  for (int i = 0; i < 5; ++i) {
    if (i % 2 == 0) {
      if (p.q_active[i]) apply(true, p.Q[i]);
    } else {
      apply(false, p.Q[i]);
    }
  }
  std::copy(T, T + 16, out);
}

}  // namespace

double gamma_ratio(const Sym& c) {
  return (std::fabs(c.q11) + std::fabs(c.q12) + 1.0) * (std::fabs(c.q12) + std::fabs(c.q22) + 1.0);
}

double ha_objective(const double abcd[16], const Sym& H) { return objective_b(blocks(abcd), H); }

int ha_search(const double abcd[16], Sym* H, double* J, std::string* err) {
  V3 h;
  int st = search(blocks(abcd), maxabs16(abcd), &h, J, err);
  if (!st) *H = hsym(h);
  return st;
}

int make_plan(const double m[16], int variant, int dispatch, const double h_fixed[3], Plan* out,
              std::string* err) {
  Plan p;
  for (int i = 0; i < 16; ++i)
    if (!std::isfinite(m[i])) {
      *err = "non-finite ABCD entry";
      return 1;
    }
  p.sym_residual = sym_residual(m);
  if (!(p.sym_residual <= kTauSym)) {
    *err = "ABCD matrix violates Eq. Intro12 (residual " + std::to_string(p.sym_residual) + ")";
    return 2;
  }
  Blocks b = blocks(m);
  double mmax = maxabs16(m);
  p.variant = variant;
  if (maxabs(b.B) <= 1e-12 * std::max(1.0, mmax)) {  // Eq. Intro20, reading R10
    p.kind = 0;
    p.Cb = b.C;
    p.Db = b.D;
    p.recomposition_residual = 0.0;
    *out = p;
    return 0;
  }
  if (variant == 3) {
    // Ding's method (Eq. Ding04/Ding12):
    //   M = (I, 0; D B^-1, I) (B, 0; 0, B^-T) (0, I; -I, 0) (I, 0; B^-1 A, I)
    // Q[0] = B^-1 A (input CM), Q[4] = D B^-1 (output CM), Db = B^-T (affine matrix).
    const double dB = det(b.B);
    if (!(std::fabs(dB) > 1e-12 * std::max(1.0, maxabs(b.B) * maxabs(b.B)))) {
      *err = "Ding's method needs det B != 0";
      return 3;
    }
    const M2 Bi = inv(b.B);
    p.kind = 3;
    p.Q[0] = symm(mul(Bi, b.A));
    p.Q[4] = symm(mul(b.D, Bi));
    p.q_active[0] = p.q_active[4] = true;
    p.Db = tr(Bi);
    p.Cb = b.C;
    // recomposition: (B Q0, B; Q4 B Q0 - B^-T, Q4 B)
    const M2 Q0 = of(p.Q[0]), Q4 = of(p.Q[4]);
    Blocks r;
    r.A = mul(b.B, Q0);
    r.B = b.B;
    r.C = sub(mul(Q4, mul(b.B, Q0)), tr(Bi));
    r.D = mul(Q4, b.B);
    double R[16];
    unblocks(r, R);
    double res = 0;
    for (int i = 0; i < 16; ++i) res = std::max(res, std::fabs(R[i] - m[i]));
    p.recomposition_residual = res;
    if (!(res <= 1e-9 * std::max(1.0, mmax))) {
      *err = "Ding recomposition check failed (residual " + std::to_string(res) + ")";
      return 3;
    }
    *out = p;
    return 0;
  }
  p.key = dispatch_key(m);
  bool form1_ = (dispatch == 1) || (p.key >= 0.0);
  double mt[16];
  if (form1_) {
    std::copy(m, m + 16, mt);
  } else {
    inverse4(m, mt);
  }
  Blocks bt = blocks(mt);
  V3 h{0, 0, 0};
  double J = kInf;
  int axis = 0;
  if (variant == 2) {
    h = {h_fixed[0], h_fixed[1], h_fixed[2]};
    J = objective_b(bt, hsym(h));
  } else if (variant == 1 && lc_choice(bt, &h, &J, &axis)) {
    // LC plan
  } else {
    int st = search(bt, mmax, &h, &J, err);
    if (st) return st;
    if (variant == 1) p.variant = 0;  // LC not applicable: HA fallback
  }
  Stages s = form1(bt, hsym(h));
  if (!s.ok) {
    *err = "det B' = 0 for the chosen H";
    return 3;
  }
  p.lc_axis = axis;
  p.H = s.H;
  p.Bp = s.Bp;
  p.P2 = s.P2;
  p.P4 = s.P4;
  p.objective = J;
  if (form1_) {
    p.kind = 1;  // CM(P4) CC(B') CM(P2) CC(H)
    p.q_active[0] = false;
    p.Q[0] = {0, 0, 0};
    p.Q[1] = negs(s.H);
    p.Q[2] = s.P2;
    p.Q[3] = negs(s.Bp);
    p.Q[4] = s.P4;
    p.q_active[2] = p.q_active[4] = true;
  } else {
    p.kind = 2;  // inverse of form I of M^-1: CC(-H~) CM(-P2~) CC(-B'~) CM(-P4~)
    p.q_active[0] = true;
    p.Q[0] = negs(s.P4);
    p.Q[1] = s.Bp;
    p.Q[2] = negs(s.P2);
    p.Q[3] = s.H;
    p.Q[4] = {0, 0, 0};
    p.q_active[2] = true;
    p.q_active[4] = false;
  }
  p.q_active[1] = p.q_active[3] = true;
  double R[16];
  chain_matrix(p, R);
  double res = 0;
  for (int i = 0; i < 16; ++i) res = std::max(res, std::fabs(R[i] - m[i]));
  p.recomposition_residual = res;
  if (!(res <= 1e-9 * std::max(1.0, mmax))) {
    *err = "recomposition check failed (residual " + std::to_string(res) + ")";
    return 3;
  }
  *out = p;
  return 0;
}

}  // namespace nslct

// Host-side planner of the NsDLCT (C++17, no CUDA).  See planner.cpp.
#pragma once
#include <cstdint>
#include <string>

namespace nslct {

struct M2 {  // 2x2 real matrix, row-major
  double a, b, c, d;
};

struct Sym {  // symmetric 2x2 (q11, q22, q12)
  double q11, q22, q12;
};

struct Plan {
  int kind = 0;           // 0 = B0, 1 = form I, 2 = form II, 3 = Ding (Eq. Ding12)
  int variant = 0;        // 0 HA, 1 LC, 2 fixed H, 3 Ding
  int lc_axis = 0;        // 0 none, 1 x, 2 y
  Sym H{}, Bp{}, P2{}, P4{};
  Sym Q[5]{};             // chirps in application order (see nslct.h)
  bool q_active[5]{};     // Q0 / Q4 may be absent
  M2 Cb{}, Db{};          // B = 0: C and D; Ding: Db = B^-T
  double objective = 0, sym_residual = 0, recomposition_residual = 0, key = 0;
};

// status codes follow nslct_status
int make_plan(const double abcd[16], int variant, int dispatch, const double h_fixed[3],
              Plan* out, std::string* err);

double gamma_ratio(const Sym& c);                 // Eq. HA16
double ha_objective(const double abcd[16], const Sym& H);  // Eq. HA24, +inf if infeasible
// HA search of reading R5: returns status, fills H and J
int ha_search(const double abcd[16], Sym* H, double* J, std::string* err);

}  // namespace nslct

// Closed-form element stiffness and its Hadamard factorisation (see element.h).
#include "element.h"

#include <cmath>

namespace tomesh {

static double fM(int a, int b) { return a == b ? 2.0 / 6.0 : 1.0 / 6.0; }
static double fS(int a, int b) { return a == b ? 1.0 : -1.0; }
static double fG(int a, int b) { (void)b; return a == 0 ? -0.5 : 0.5; }  // int N_a' N_b

// I(p,q) = int d_p N_A d_q N_B over the unit cell.
static double integ(int dim, int A, int B, int p, int q) {
  double v = 1.0;
  for (int k = 0; k < dim; ++k) {
    int a = (A >> k) & 1, b = (B >> k) & 1;
    if (k == p && k == q) v *= fS(a, b);
    else if (k == p) v *= fG(a, b);
    else if (k == q) v *= fG(b, a);
    else v *= fM(a, b);
  }
  return v;
}

void build_K0(int dim, double nu, double *K) {
  const double mu = 1.0 / (2.0 * (1.0 + nu));
  const double lam = (dim == 2) ? nu / (1.0 - nu * nu) : nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const int nc = 1 << dim, n = dim * nc;
  for (int A = 0; A < nc; ++A)
    for (int i = 0; i < dim; ++i)
      for (int B = 0; B < nc; ++B)
        for (int j = 0; j < dim; ++j) {
          double v = lam * integ(dim, A, B, i, j) + mu * integ(dim, A, B, j, i);
          if (i == j)
            for (int k = 0; k < dim; ++k) v += mu * integ(dim, A, B, k, k);
          K[(dim * A + i) * n + dim * B + j] = v;
        }
}

int build_K0_hadamard(double nu, K0Had3 *out) {
  double K[24 * 24];
  build_K0(3, nu, K);
  auto H = [](int m, int a) { return (__builtin_popcount(m & a) & 1) ? -1.0 : 1.0; };
  // Khat[(m,i),(n,j)] = sum_{a,b} H(m,a) K[(a,i),(b,j)] H(n,b) / 64
  double Kh[24][24];
  for (int m = 0; m < 8; ++m)
    for (int i = 0; i < 3; ++i)
      for (int n = 0; n < 8; ++n)
        for (int j = 0; j < 3; ++j) {
          double s = 0.0;
          for (int a = 0; a < 8; ++a)
            for (int b = 0; b < 8; ++b) s += H(m, a) * K[(3 * a + i) * 24 + 3 * b + j] * H(n, b);
          Kh[3 * m + i][3 * n + j] = s / 64.0;
        }
  double scale = 0.0;
  for (int r = 0; r < 24; ++r)
    for (int c = 0; c < 24; ++c) scale = std::fmax(scale, std::fabs(Kh[r][c]));
  int bad = 0;
  for (int m = 0; m < 8; ++m)
    for (int i = 0; i < 3; ++i)
      for (int n = 0; n < 8; ++n)
        for (int j = 0; j < 3; ++j) {
          double v = Kh[3 * m + i][3 * n + j];
          bool expected;
          if (i == j) expected = (m == n);
          else expected = (((m >> i) & 1) != ((m >> j) & 1)) && (n == (m ^ ((1 << i) | (1 << j))));
          if (!expected && std::fabs(v) > 1e-13 * scale) ++bad;
        }
  for (int i = 0; i < 3; ++i)
    for (int m = 0; m < 8; ++m) {
      out->diag[i][m] = Kh[3 * m + i][3 * m + i];
      for (int j = 0; j < 3; ++j) {
        if (j == i || ((m >> i) & 1) == ((m >> j) & 1)) {
          out->off[i][j][m] = 0.0;
        } else {
          int n = m ^ ((1 << i) | (1 << j));
          out->off[i][j][m] = Kh[3 * m + i][3 * n + j];
        }
      }
    }
  // exact zeros where the factorisation says so (mode 0 is the rigid translation)
  for (int i = 0; i < 3; ++i) out->diag[i][0] = 0.0;
  return bad;
}

int build_K0_hadamard_sym(const K0Had3 &h, K0HadSym *out) {
  auto pop = [](int m) { return (m & 1) + ((m >> 1) & 1) + ((m >> 2) & 1); };
  bool set_d[2][3] = {}, set_o[2][2] = {};
  for (int i = 0; i < 3; ++i)
    for (int m = 1; m < 8; ++m) {
      const int b = (m >> i) & 1, n = pop(m) - b;
      if (!set_d[b][n]) { out->d[b][n] = h.diag[i][m]; set_d[b][n] = true; }
      for (int j = 0; j < 3; ++j) {
        if (j == i || ((m >> j) & 1) == b) continue;
        const int t = ((m >> (3 - i - j)) & 1);
        if (!set_o[b][t]) { out->o[b][t] = h.off[i][j][m]; set_o[b][t] = true; }
      }
    }
  out->d[0][0] = 0.0;
  int bad = 0;
  auto differs = [](double a, double c) { return std::fabs(a - c) > 1e-15 * std::fmax(std::fabs(c), 1e-300); };
  for (int i = 0; i < 3; ++i)
    for (int m = 1; m < 8; ++m) {
      const int b = (m >> i) & 1, n = pop(m) - b;
      if (differs(h.diag[i][m], out->d[b][n])) ++bad;
      for (int j = 0; j < 3; ++j) {
        if (j == i || ((m >> j) & 1) == b) continue;
        if (differs(h.off[i][j][m], out->o[b][(m >> (3 - i - j)) & 1])) ++bad;
      }
    }
  return bad;
}

}  // namespace tomesh

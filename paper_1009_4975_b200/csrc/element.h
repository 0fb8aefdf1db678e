// Element stiffness of the bi/tri-linear displacement element
// in closed form, and its Walsh-Hadamard (tensor-sign) factorisation used by
// the 3D operator kernels.
//
// Closed form (E = 1, edge h = 1; unit thickness and plane stress in 2D):
//   K[(a,i),(b,j)] = lam I(i,j) + mu I(j,i) + mu delta_ij sum_k I(k,k)
//   I(p,q) = int d_p N_a d_q N_b = prod_k f_k,  with the 1D factors
//     f_k = S(a_k,b_k) if k == p == q,   S = [1 -1; -1 1]
//           G(a_k,b_k) if k == p != q,   G = 1/2 [-1 -1; 1 1]   (int N_a' N_b)
//           G(b_k,a_k) if k == q != p,
//           M(a_k,b_k) otherwise,        M = 1/6 [2 1; 1 2]
//   lam = E nu/((1+nu)(1-2nu)) in 3D, E nu/(1-nu^2) in plane stress;
//   mu = E/(2(1+nu)).  K0(h) = h^(d-2) K0(1).
// This is a different derivation from the oracle's Gauss quadrature; the two
// are compared entry by entry in tests/test_host_lib.py.
//
// Hadamard form: with H = [1 1; 1 -1] per axis, H M H = diag(1, 1/3),
// H S H = diag(0, 4), H G H = -2 e1 e0^T.  So Khat = H3 K H3 is block-sparse:
// each 8x8 component block (i,i) is diagonal and each (i,j != i) block has
// one nonzero per mode m with m_i != m_j, at column mode m ^ (e_i | e_j).
// y = K x = H3 Khat H3 x / 64, so the dense 24x24 product (576 FMA) becomes
// 2 x 72 add/sub + 21 + 24 multiply-adds.
#pragma once

namespace tomesh {

struct K0Dense2 { double K[8 * 8]; };
struct K0Dense3 { double K[24 * 24]; };

// Hadamard-basis coefficients for H8, already divided by 64.
//   diag[i][m]     coefficient of xhat[(m,i)] in yhat[(m,i)]
//   off[i][j][m]   coefficient of xhat[(m ^ (e_i|e_j), j)] in yhat[(m,i)]
//                  (zero unless bit i of m != bit j of m)
struct K0Had3 {
  double diag[3][8];
  double off[3][3][8];
};

// The 45 nonzero Hadamard coefficients take only 9 distinct values:
//   diag[i][m] = d[b][n],  b = bit i of m, n = number of the other bits of m set
//                (d[0][0] = 0: the rigid translation mode);
//   off[i][j][m] = o[b][t], b = bit i of m (bit j differs), t = bit 3-i-j of m.
// (Per axis the Hadamard images of the 1D mass, stiffness and gradient
// matrices are diag(1, 1/3), diag(0, 4) and -2 e1 e0^T, so every coefficient
// is a product of these per-axis factors with lambda or mu.)
struct K0HadSym {
  double d[2][3];
  double o[2][2];
};

void build_K0(int dim, double nu, double *K);      // E = 1, h = 1
// Class values of `h`; returns the number of coefficients that differ from
// their class value by more than 1e-15 relative (0 expected).
int build_K0_hadamard_sym(const K0Had3 &h, K0HadSym *out);
int build_K0_hadamard(double nu, K0Had3 *out);     // returns 0 if the structure check passes

}  // namespace tomesh

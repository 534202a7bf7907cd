// =============================================================================
// egfem_oracle.cpp — plain, slow, obviously-correct CPU oracle for the EGFEM hot
// path (arXiv 2005.06193).  TEST INFRASTRUCTURE ONLY: it may be loaded solely by
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// legs.  It shares no code, header, table or constant generator with the CUDA
// path (paper_2005_06193_b200/csrc) and neither side includes the other.
//
// Everything is fp64, sequential, in the paper's order.  It runs single-threaded unless
// oracle_set_threads(n > 1) is called (only bench.py's all-cores cpu_baseline timing does):
// then the row loops of apply / jacobian and the cell loops of interp are split across OpenMP
// threads, every row (cell) still computed alone and in its sequential order, so the results
// are bitwise those of one thread.
//   * T_ijk = ∫ (slot_a φ_i)(slot_b φ_j)(slot_c η_k) dx assembled element by
//     element with a quadrature rule (eq. (egfem_terms);
//     L253 K_a; L327 M; L400 N), duplicates summed in emission order, stored as
//     SPEC's lexicographically sorted COO.
//   * w = f(Π_u u, Π_∇u ·₂ u) pointwise at the W-DOFs (PAPER.md L96–99 eq.
//     (egfem_coeffs), L153–169 §3.2).
//   * r = T:(u⊗w), r_i = Σ_jk T_ijk u_j w_k.
//   * A = T·w and the Newton Jacobian
//     J = T·w + (T·₂u)·D_u w, the Schur complement of the block Jacobian of
//     PAPER.md L290 (reading C10 in DESIGN.md), formed as a literal sparse
//     block product.
//
// Pinned by tests/test_oracle_*.py (closed forms, brute force, partition of unity,
// symmetry, Euler homogeneity, finite differences, Case-1 exactness).
// =============================================================================
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <numeric>
#include <vector>

namespace {

enum { OF_P0 = 0, OF_P1 = 1, OF_P2 = 2, OF_QUAD = 3 };  // QUAD: I_k of PAPER.md L117–139
enum { OFORM_CONV_K = 0, OFORM_CONV_J = 1, OFORM_PLAP = 2, OFORM_MASS3 = 3, OFORM_CONV_I = 4 };
enum { OK_IDENTITY = 0, OK_SQUARE = 1, OK_GRADPOW_P0 = 2, OK_P1_TO_P2_SQUARE = 3, OK_MINSURF_P0 = 4, OK_RECIPROCAL = 5 };
enum { OJ_PICARD = 0, OJ_NEWTON = 1 };

// Slot operators: which functional of a basis function enters a slot.
enum { OP_VALUE = 0, OP_DX = 1, OP_DXDY = 2, OP_GRAD = 3 };

struct Space {
  int family;
  int64_t n_dofs;
  int n_loc;
  std::vector<int32_t> cell_dofs;  // n_cells * n_loc
};

struct OTensor {
  // mesh
  int dim;
  int64_t n_vertices, n_cells;
  std::vector<double> coords;
  std::vector<int32_t> cells;
  Space V, W;
  int form;
  int64_t row_begin, row_end;
  // canonical tensor (rows outside [row_begin,row_end) are empty)
  std::vector<int64_t> t_row_ptr;
  std::vector<int32_t> t_j, t_k;
  std::vector<double> t_val;
  // CSR pattern (union of element cliques over V-DOFs)
  std::vector<int64_t> csr_row_ptr;
  std::vector<int32_t> csr_col;
  // W = QUAD: barycentric coordinates of the quadrature points (the W DOFs of each cell)
  std::vector<double> wbary;
};

// ---------------------------------------------------------------- geometry
// Affine map x = x0 + B ξ with B = [x1-x0, ..., xd-x0]; ∇λ_{1..d} are the rows of
// B^{-1} and ∇λ_0 = -Σ_{a≥1} ∇λ_a; |K| = |det B| / d!.
struct Geo {
  double grad[4][3];  // grad[a][x]
  double vol;
};

static double det3(const double m[3][3]) {
  return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1])
       - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0])
       + m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

static Geo geometry(const OTensor& T, int64_t cell) {
  Geo g;
  std::memset(&g, 0, sizeof(g));
  const int d = T.dim;
  const int32_t* cv = &T.cells[cell * (d + 1)];
  double B[3][3] = {{0}};
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < d; ++c)
      B[r][c] = T.coords[(int64_t)cv[c + 1] * d + r] - T.coords[(int64_t)cv[0] * d + r];
  double Binv[3][3] = {{0}};
  double det = 0;
  if (d == 1) {
    det = B[0][0];
    Binv[0][0] = 1.0 / det;
  } else if (d == 2) {
    det = B[0][0] * B[1][1] - B[0][1] * B[1][0];
    Binv[0][0] = B[1][1] / det;
    Binv[0][1] = -B[0][1] / det;
    Binv[1][0] = -B[1][0] / det;
    Binv[1][1] = B[0][0] / det;
  } else {
    det = det3(B);
    // inverse = adj(B)/det, adj = transpose of cofactor matrix
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        int r1 = (c + 1) % 3, r2 = (c + 2) % 3, c1 = (r + 1) % 3, c2 = (r + 2) % 3;
        Binv[r][c] = (B[r1][c1] * B[r2][c2] - B[r1][c2] * B[r2][c1]) / det;
      }
  }
  double fact = (d == 1) ? 1.0 : (d == 2 ? 2.0 : 6.0);
  g.vol = std::fabs(det) / fact;
  for (int a = 1; a <= d; ++a)
    for (int x = 0; x < d; ++x) g.grad[a][x] = Binv[a - 1][x];
  for (int x = 0; x < d; ++x) {
    double s = 0;
    for (int a = 1; a <= d; ++a) s += g.grad[a][x];
    g.grad[0][x] = -s;
  }
  return g;
}

// ---------------------------------------------------------------- bases
// Lagrange bases in barycentric coordinates λ (dim+1 entries).
// P0: 1.  P1: λ_a.  P2 (2D only, local order v0,v1,v2,m01,m12,m20):
//   vertex a: λ_a(2λ_a-1),  midpoint (a,b): 4 λ_a λ_b.
static void basis(int family, int d, const double* lam, const Geo& g, int n_loc,
                  double* val, double (*grad)[3]) {
  for (int l = 0; l < n_loc; ++l) {
    val[l] = 0;
    for (int x = 0; x < 3; ++x) grad[l][x] = 0;
  }
  if (family == OF_P0) {
    val[0] = 1.0;
  } else if (family == OF_P1) {
    for (int a = 0; a <= d; ++a) {
      val[a] = lam[a];
      for (int x = 0; x < d; ++x) grad[a][x] = g.grad[a][x];
    }
  } else {  // P2, d == 2
    for (int a = 0; a < 3; ++a) {
      val[a] = lam[a] * (2 * lam[a] - 1);
      for (int x = 0; x < d; ++x) grad[a][x] = (4 * lam[a] - 1) * g.grad[a][x];
    }
    const int ea[3] = {0, 1, 2}, eb[3] = {1, 2, 0};
    for (int m = 0; m < 3; ++m) {
      int a = ea[m], b = eb[m];
      val[3 + m] = 4 * lam[a] * lam[b];
      for (int x = 0; x < d; ++x) grad[3 + m][x] = 4 * (lam[a] * g.grad[b][x] + lam[b] * g.grad[a][x]);
    }
  }
}

static int family_degree(int f) { return (f == OF_P0 || f == OF_QUAD) ? 0 : (f == OF_P1 ? 1 : 2); }

// ---------------------------------------------------------------- quadrature
// Reference rules in barycentric coordinates, weights summing to 1 (physical
// weight = weight × |K|).  1D: 3-point Gauss.  2D: centroid (deg 1),
// (2/3,1/6,1/6) (deg 2), 6-point symmetric Dunavant (deg 4).  3D: centroid,
// 4-point (deg 2), collapsed Gauss product (deg ≥ 3, below).
struct Rule {
  int nq;
  std::vector<double> bary;  // nq*(d+1)
  std::vector<double> w;
};

// n-point Gauss–Legendre on [0,1] (textbook: Newton on the three-term Legendre recurrence
// P_{m+1} = ((2m+1) x P_m − m P_{m−1})/(m+1) on [−1,1], weights 2/((1−x²)P_n'(x)²), then
// mapped to [0,1]).  Exact for polynomials of degree ≤ 2n−1.
static void gauss_legendre01(int n, std::vector<double>& x01, std::vector<double>& w01) {
  const double pi = std::acos(-1.0);
  x01.assign(n, 0.0);
  w01.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double x = std::cos(pi * (i + 0.75) / (n + 0.5));
    double dp = 0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int m = 1; m < n; ++m) {
        double p2 = ((2.0 * m + 1.0) * x * p1 - m * p0) / (m + 1.0);
        p0 = p1;
        p1 = p2;
      }
      // p1 = P_n(x), p0 = P_{n-1}(x)
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-17) break;
    }
    x01[i] = 0.5 * (1.0 - x);
    w01[i] = 0.5 * 2.0 / ((1.0 - x * x) * dp * dp);
  }
}

// Tetrahedral rule exact for total degree `degree` (≥ 3): the collapsed-coordinate (Duffy)
// product of Gauss–Legendre rules.  The unit cube maps onto the reference tetrahedron
// {ξ ≥ 0, ξ1+ξ2+ξ3 ≤ 1} by ξ1 = s, ξ2 = t(1−s), ξ3 = v(1−s)(1−t) with Jacobian (1−s)²(1−t); a
// polynomial of degree p in ξ becomes one of degree ≤ p+2 in s, p+1 in t, p in v, so n points
// per direction with 2n−1 ≥ p+2 integrate it exactly.  All weights are positive.  Weights are
// normalised to sum to 1 (physical weight = weight × |K|), barycentric λ = (1−Σξ, ξ1, ξ2, ξ3).
// This makes every 3D form the exact integral of PAPER.md L196–203 eq. (egfem_terms), e.g. the
// trilinear mass M of L327 (degree 3 for P1×P1×P1).
static Rule collapsed_gauss_tet(int degree) {
  const int n = (degree + 4) / 2;
  std::vector<double> x, w;
  gauss_legendre01(n, x, w);
  Rule R;
  R.nq = n * n * n;
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b)
      for (int c = 0; c < n; ++c) {
        const double s = x[a], t = x[b], v = x[c];
        const double xi1 = s, xi2 = t * (1 - s), xi3 = v * (1 - s) * (1 - t);
        R.bary.push_back(1.0 - xi1 - xi2 - xi3);
        R.bary.push_back(xi1);
        R.bary.push_back(xi2);
        R.bary.push_back(xi3);
        R.w.push_back(6.0 * w[a] * w[b] * w[c] * (1 - s) * (1 - s) * (1 - t));
      }
  return R;
}

static Rule default_rule(int d, int degree) {
  Rule R;
  if (d == 1) {
    double s = std::sqrt(3.0 / 5.0);
    double xi[3] = {(1 - s) / 2, 0.5, (1 + s) / 2};
    double w[3] = {5.0 / 18, 8.0 / 18, 5.0 / 18};
    R.nq = 3;
    for (int q = 0; q < 3; ++q) {
      R.bary.push_back(1 - xi[q]);
      R.bary.push_back(xi[q]);
      R.w.push_back(w[q]);
    }
    return R;
  }
  if (d == 2) {
    if (degree <= 1) {
      R.nq = 1;
      R.bary = {1.0 / 3, 1.0 / 3, 1.0 / 3};
      R.w = {1.0};
    } else if (degree <= 2) {
      R.nq = 3;
      R.bary = {2.0 / 3, 1.0 / 6, 1.0 / 6, 1.0 / 6, 2.0 / 3, 1.0 / 6, 1.0 / 6, 1.0 / 6, 2.0 / 3};
      R.w = {1.0 / 3, 1.0 / 3, 1.0 / 3};
    } else {
      // Two S21 orbits (a, a, 1-2a): degree-4 exact (reading C3).
      const double a1 = 0.445948490915965, w1 = 0.2233815896780118;
      const double a2 = 0.091576213509770549, w2 = 0.10995174365532154;
      const double A[2] = {a1, a2}, W[2] = {w1, w2};
      R.nq = 6;
      for (int o = 0; o < 2; ++o) {
        double a = A[o], b = 1 - 2 * a;
        double pts[3][3] = {{b, a, a}, {a, b, a}, {a, a, b}};
        for (int q = 0; q < 3; ++q) {
          for (int x = 0; x < 3; ++x) R.bary.push_back(pts[q][x]);
          R.w.push_back(W[o]);
        }
      }
    }
    return R;
  }
  // d == 3
  if (degree <= 1) {
    R.nq = 1;
    R.bary = {0.25, 0.25, 0.25, 0.25};
    R.w = {1.0};
  } else if (degree == 2) {
    const double a = 0.1381966011250105, b = 0.5854101966249685;
    R.nq = 4;
    for (int q = 0; q < 4; ++q)
      for (int x = 0; x < 4; ++x) R.bary.push_back(x == q ? b : a);
    R.w = {0.25, 0.25, 0.25, 0.25};
  } else {
    R = collapsed_gauss_tet(degree);
  }
  return R;
}

// Slot operators of each form, slot order (i, j, k) = (test, u-slot, w-slot).
static void form_ops(int form, int* opA, int* opB, int* opC) {
  switch (form) {
    case OFORM_CONV_K: *opA = OP_VALUE; *opB = OP_VALUE; *opC = OP_DX; break;    // ∫ φ_i φ_j ∂x φ_k
    case OFORM_CONV_J: *opA = OP_VALUE; *opB = OP_DXDY; *opC = OP_VALUE; break;  // ∫ φ_i (∂x+∂y)φ_j φ_k
    case OFORM_PLAP:   *opA = OP_GRAD;  *opB = OP_GRAD; *opC = OP_VALUE; break;  // ∫ ψ_k ∇φ_i·∇φ_j
    case OFORM_MASS3:  *opA = OP_VALUE; *opB = OP_VALUE; *opC = OP_VALUE; break; // ∫ φ_i φ_j η_k
    default:           *opA = OP_DXDY;  *opB = OP_VALUE; *opC = OP_VALUE; break; // ∫ (∂x+∂y)φ_i φ_j φ_k (paper N)
  }
}

static int op_degree(int op, int fam) {
  int d = family_degree(fam);
  if (op == OP_VALUE) return d;
  return d > 0 ? d - 1 : 0;
}

static double apply_op(int op, int d, double val, const double* grad) {
  if (op == OP_VALUE) return val;
  if (op == OP_DX) return grad[0];
  // (∂x + ∂y): sum of the first min(d,2) partial derivatives
  double s = grad[0];
  if (d >= 2) s += grad[1];
  return s;
}

}  // namespace

extern "C" {

typedef struct OTensor OTensor_t;

// Build the canonical tensor.  Returns 0 on success, negative on bad input.
int oracle_build(int dim, int64_t n_vertices, const double* coords, int64_t n_cells,
                 const int32_t* cells, int v_family, int64_t v_ndofs, int v_nloc,
                 const int32_t* v_cell_dofs, int w_family, int64_t w_ndofs, int w_nloc,
                 const int32_t* w_cell_dofs, int form, int nq, const double* qbary,
                 const double* qw, int64_t row_begin, int64_t row_end, void** out) {
  if (dim < 1 || dim > 3) return -1;
  if (v_family == OF_P2 && dim != 2) return -2;
  if (w_family == OF_P2 && dim != 2) return -2;
  OTensor* T = new OTensor();
  T->dim = dim;
  T->n_vertices = n_vertices;
  T->n_cells = n_cells;
  T->coords.assign(coords, coords + n_vertices * dim);
  T->cells.assign(cells, cells + n_cells * (dim + 1));
  T->V = {v_family, v_ndofs, v_nloc, std::vector<int32_t>(v_cell_dofs, v_cell_dofs + n_cells * v_nloc)};
  T->W = {w_family, w_ndofs, w_nloc, std::vector<int32_t>(w_cell_dofs, w_cell_dofs + n_cells * w_nloc)};
  T->form = form;
  if (row_begin < 0) row_begin = 0;
  if (row_end < 0 || row_end > v_ndofs) row_end = v_ndofs;
  T->row_begin = row_begin;
  T->row_end = row_end;

  int opA, opB, opC;
  form_ops(form, &opA, &opB, &opC);
  if (form == OFORM_PLAP && w_family != OF_P0 && nq <= 0) {
    // PLAP with a non-P0 W still follows the quadrature definition below.
  }
  Rule R;
  if (nq > 0) {
    R.nq = nq;
    R.bary.assign(qbary, qbary + nq * (dim + 1));
    R.w.assign(qw, qw + nq);
  } else if (w_family == OF_QUAD) {
    // I_k: the W DOFs are the points of the assembly rule itself; take the
    // default rule with exactly w_nloc points.
    bool found = false;
    for (int deg : {1, 2, 4, 5}) {
      R = default_rule(dim, deg);
      if (R.nq == w_nloc) {
        found = true;
        break;
      }
    }
    if (!found) {
      delete T;
      return -4;
    }
  } else {
    int deg = op_degree(opA, v_family) + op_degree(opB, v_family) + op_degree(opC, w_family);
    if (opA == OP_GRAD) deg = 2 * op_degree(OP_GRAD, v_family) + op_degree(opC, w_family);
    R = default_rule(dim, deg);
  }
  if (w_family == OF_QUAD) {
    if (R.nq != w_nloc || opC != OP_VALUE) {
      delete T;
      return -5;
    }
    T->wbary = R.bary;
  }

  // ---- emit every local triple, cell-major then (a,b,c) lexicographic
  struct Trip { int32_t i, j, k; double v; };
  std::vector<Trip> trips;
  const int nA = v_nloc, nC = w_nloc;
  std::vector<double> vv(nA), wv(nC), Tk(nA * nA * nC);
  std::vector<double> vg(nA * 3), wg(nC * 3);
  for (int64_t K = 0; K < n_cells; ++K) {
    const int32_t* I = &T->V.cell_dofs[K * nA];
    const int32_t* Wd = &T->W.cell_dofs[K * nC];
    bool any = false;
    for (int a = 0; a < nA; ++a) any |= (I[a] >= row_begin && I[a] < row_end);
    if (!any) continue;
    Geo g = geometry(*T, K);
    std::fill(Tk.begin(), Tk.end(), 0.0);
    for (int q = 0; q < R.nq; ++q) {
      const double* lam = &R.bary[q * (dim + 1)];
      basis(v_family, dim, lam, g, nA, vv.data(), reinterpret_cast<double(*)[3]>(vg.data()));
      if (w_family == OF_QUAD) {  // η_ℓ = w_ℓ δ_{x_ℓ}: ∫ v η_ℓ = w_ℓ v(x_ℓ)
        for (int c = 0; c < nC; ++c) {
          wv[c] = (c == q) ? 1.0 : 0.0;
          wg[c * 3] = wg[c * 3 + 1] = wg[c * 3 + 2] = 0.0;
        }
      } else {
        basis(w_family, dim, lam, g, nC, wv.data(), reinterpret_cast<double(*)[3]>(wg.data()));
      }
      double wq = R.w[q] * g.vol;
      for (int a = 0; a < nA; ++a)
        for (int b = 0; b < nA; ++b)
          for (int c = 0; c < nC; ++c) {
            double fab;
            if (opA == OP_GRAD) {
              fab = 0;
              for (int x = 0; x < dim; ++x) fab += vg[a * 3 + x] * vg[b * 3 + x];
            } else {
              fab = apply_op(opA, dim, vv[a], &vg[a * 3]) * apply_op(opB, dim, vv[b], &vg[b * 3]);
            }
            double fc = apply_op(opC, dim, wv[c], &wg[c * 3]);
            Tk[(a * nA + b) * nC + c] += wq * fab * fc;
          }
    }
    for (int a = 0; a < nA; ++a) {
      if (I[a] < row_begin || I[a] >= row_end) continue;
      for (int b = 0; b < nA; ++b)
        for (int c = 0; c < nC; ++c) trips.push_back({I[a], I[b], Wd[c], Tk[(a * nA + b) * nC + c]});
    }
  }

  // ---- canonicalise: stable sort by (i,j,k), sum duplicates in emission order
  std::vector<int64_t> order(trips.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
    const Trip& A = trips[x];
    const Trip& B = trips[y];
    if (A.i != B.i) return A.i < B.i;
    if (A.j != B.j) return A.j < B.j;
    return A.k < B.k;
  });
  T->t_row_ptr.assign(v_ndofs + 1, 0);
  for (size_t s = 0; s < order.size();) {
    const Trip& A = trips[order[s]];
    double sum = 0;
    size_t e = s;
    while (e < order.size() && trips[order[e]].i == A.i && trips[order[e]].j == A.j &&
           trips[order[e]].k == A.k) {
      sum += trips[order[e]].v;
      ++e;
    }
    T->t_j.push_back(A.j);
    T->t_k.push_back(A.k);
    T->t_val.push_back(sum);
    T->t_row_ptr[A.i + 1]++;
    s = e;
  }
  for (int64_t i = 0; i < v_ndofs; ++i) T->t_row_ptr[i + 1] += T->t_row_ptr[i];

  // ---- CSR pattern: union over cells of (I[a], I[b]), sorted and unique per row
  std::vector<std::pair<int32_t, int32_t>> pairs;
  for (int64_t K = 0; K < n_cells; ++K) {
    const int32_t* I = &T->V.cell_dofs[K * nA];
    for (int a = 0; a < nA; ++a) {
      if (I[a] < row_begin || I[a] >= row_end) continue;
      for (int b = 0; b < nA; ++b) pairs.push_back({I[a], I[b]});
    }
  }
  std::sort(pairs.begin(), pairs.end());
  pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
  T->csr_row_ptr.assign(v_ndofs + 1, 0);
  for (auto& pr : pairs) {
    T->csr_col.push_back(pr.second);
    T->csr_row_ptr[pr.first + 1]++;
  }
  for (int64_t i = 0; i < v_ndofs; ++i) T->csr_row_ptr[i + 1] += T->csr_row_ptr[i];
  *out = T;
  return 0;
}

void oracle_free(void* h) { delete static_cast<OTensor*>(h); }

// The default rule the element loop takes for (dim, integrand degree): returns the number of
// points and, if the buffers are non-NULL (capacity `cap` points), its barycentric points and
// weights.  Exported so tests can pin every rule by monomial exactness.
int oracle_rule(int dim, int degree, int cap, double* bary, double* w) {
  if (dim < 1 || dim > 3) return -1;
  Rule R = default_rule(dim, degree);
  if (bary && w) {
    if (R.nq > cap) return -2;
    std::copy(R.bary.begin(), R.bary.end(), bary);
    std::copy(R.w.begin(), R.w.end(), w);
  }
  return R.nq;
}

void oracle_sizes(const void* h, int64_t* nnz, int64_t* nnz_csr, int64_t* n_u, int64_t* n_f) {
  const OTensor* T = static_cast<const OTensor*>(h);
  *nnz = (int64_t)T->t_val.size();
  *nnz_csr = (int64_t)T->csr_col.size();
  *n_u = T->V.n_dofs;
  *n_f = T->W.n_dofs;
}

static int64_t csr_find(const OTensor* T, int64_t i, int32_t col) {
  const int32_t* b = T->csr_col.data() + T->csr_row_ptr[i];
  const int32_t* e = T->csr_col.data() + T->csr_row_ptr[i + 1];
  const int32_t* p = std::lower_bound(b, e, col);
  if (p == e || *p != col) return -1;
  return p - T->csr_col.data();
}

// Export canonical arrays (NULL = skip).  slot_ik only for W == V numbering,
// loc only for P0 W (bits 0-1: local index of i in cell k, bits 2-3: of j).
int oracle_export(const void* h, int64_t* t_row_ptr, int32_t* t_j, int32_t* t_k, double* t_val,
                  int64_t* csr_row_ptr, int32_t* csr_col, int32_t* slot_ij, int32_t* slot_ik,
                  uint8_t* loc) {
  const OTensor* T = static_cast<const OTensor*>(h);
  size_t nnz = T->t_val.size();
  if (t_row_ptr) std::copy(T->t_row_ptr.begin(), T->t_row_ptr.end(), t_row_ptr);
  if (t_j) std::copy(T->t_j.begin(), T->t_j.end(), t_j);
  if (t_k) std::copy(T->t_k.begin(), T->t_k.end(), t_k);
  if (t_val) std::copy(T->t_val.begin(), T->t_val.end(), t_val);
  if (csr_row_ptr) std::copy(T->csr_row_ptr.begin(), T->csr_row_ptr.end(), csr_row_ptr);
  if (csr_col) std::copy(T->csr_col.begin(), T->csr_col.end(), csr_col);
  std::vector<int64_t> wcell;  // cell-wise W (P0: one DOF per cell; QUAD: N_q per cell)
  if (loc) {
    wcell.assign(T->W.n_dofs, -1);
    for (int64_t K = 0; K < T->n_cells; ++K)
      for (int l = 0; l < T->W.n_loc; ++l) wcell[T->W.cell_dofs[K * T->W.n_loc + l]] = K;
  }
  for (int64_t i = 0; i < T->V.n_dofs; ++i) {
    for (int64_t e = T->t_row_ptr[i]; e < T->t_row_ptr[i + 1]; ++e) {
      if (slot_ij) {
        int64_t s = csr_find(T, i, T->t_j[e]);
        if (s < 0) return -3;
        slot_ij[e] = (int32_t)s;
      }
      if (slot_ik) {
        int64_t s = csr_find(T, i, T->t_k[e]);
        if (s < 0) return -4;
        slot_ik[e] = (int32_t)s;
      }
      if (loc) {
        const int64_t cell = wcell[T->t_k[e]];  // the cell owning W-DOF t_k[e]
        if (cell < 0) return -5;
        const int32_t* cv = &T->V.cell_dofs[cell * T->V.n_loc];
        int li = -1, lj = -1;
        for (int a = 0; a < T->V.n_loc; ++a) {
          if (cv[a] == i) li = a;
          if (cv[a] == T->t_j[e]) lj = a;
        }
        if (li < 0 || lj < 0) return -5;
        loc[e] = (uint8_t)(li | (lj << 2));
      }
    }
  }
  (void)nnz;
  return 0;
}

// ---------------------------------------------------------------- interp
// w = f(Π_u u, Π_∇u ·₂ u) at the W-DOFs.
//   IDENTITY:        f(u) = u,  W = V  (GFEM, Π_u = identity, L338)
//   SQUARE:          f(u) = u², W = V  (L336 with Π = identity)
//   GRADPOW_P0:      f(∇u) = ‖∇u‖^{p-2} at the P0 DOF of each cell (L574, L582)
//   P1_TO_P2_SQUARE: f(u) = u² at the P2 DOFs, w = (Π_u u) ⊙ (Π_u u) (L336)
//   MINSURF_P0:      a(∇u) = (1 + ‖∇u‖²)^{-1/2} at the P0 DOF of each cell (minimal surface, L605, L609)
//   RECIPROCAL:      c̃(u) = σ/(k + u) with σ = 1, k = p (biochemical, L520–535) at the W-DOFs:
//                    the nodes (W = V) or the cell centroid (W = P0, V = P1: u_h(x_K) = Σ_a u_a λ_a(x_K))
// Work items [c0, c1): cells for the cell-wise kinds, W-DOFs for the nodal ones (c1 < 0: all).
int oracle_interp_range(const void* h, int kind, double p, const double* u, double* w, int64_t c0, int64_t c1) {
  const OTensor* T = static_cast<const OTensor*>(h);
  const int d = T->dim;
  const bool nodal = (kind == OK_IDENTITY || kind == OK_SQUARE ||
                      (kind == OK_RECIPROCAL && T->W.family == T->V.family && T->W.n_dofs == T->V.n_dofs)) &&
                     T->W.family != OF_QUAD;
  const int64_t n_items = nodal ? T->W.n_dofs : T->n_cells;
  if (c1 < 0 || c1 > n_items) c1 = n_items;
  if (c0 < 0) c0 = 0;
  if (T->W.family == OF_QUAD && (kind == OK_SQUARE || kind == OK_RECIPROCAL)) {
    // Case 3: f evaluated at the quadrature points, u_h(x_ℓ) = Σ_a λ_a(x_ℓ) u_a
    if (T->V.family != OF_P1) return -2;
    const int nq = T->W.n_loc;
    for (int64_t K = c0; K < c1; ++K) {
      const int32_t* I = &T->V.cell_dofs[K * T->V.n_loc];
      for (int l = 0; l < nq; ++l) {
        double uh = 0;
        for (int a = 0; a <= d; ++a) uh += T->wbary[l * (d + 1) + a] * u[I[a]];
        w[T->W.cell_dofs[K * nq + l]] = (kind == OK_SQUARE) ? uh * uh : 1.0 / (p + uh);
      }
    }
    return 0;
  }
  if (kind == OK_IDENTITY || kind == OK_SQUARE) {
    if (T->W.n_dofs != T->V.n_dofs) return -1;
    for (int64_t k = c0; k < c1; ++k) w[k] = (kind == OK_IDENTITY) ? u[k] : u[k] * u[k];
    return 0;
  }
  if (kind == OK_RECIPROCAL) {
    if (T->W.family == T->V.family && T->W.n_dofs == T->V.n_dofs) {
      for (int64_t k = c0; k < c1; ++k) w[k] = 1.0 / (p + u[k]);
      return 0;
    }
    if (T->W.family != OF_P0 || T->V.family != OF_P1) return -2;
    for (int64_t K = c0; K < c1; ++K) {
      const int32_t* I = &T->V.cell_dofs[K * T->V.n_loc];
      double uc = 0;  // u_h at the centroid: λ_a = 1/(d+1)
      for (int a = 0; a <= d; ++a) uc += u[I[a]] / (d + 1);
      w[T->W.cell_dofs[K]] = 1.0 / (p + uc);
    }
    return 0;
  }
  if (kind == OK_MINSURF_P0) {
    if ((T->W.family != OF_P0 && T->W.family != OF_QUAD) || T->V.family != OF_P1) return -2;
#pragma omp parallel for schedule(static)
    for (int64_t K = c0; K < c1; ++K) {
      Geo g = geometry(*T, K);
      const int32_t* I = &T->V.cell_dofs[K * T->V.n_loc];
      double gu[3] = {0, 0, 0};  // (Π_∇u ·₂ u) at the cell's DOF
      for (int a = 0; a <= d; ++a)
        for (int x = 0; x < d; ++x) gu[x] += u[I[a]] * g.grad[a][x];
      double gg = 0;
      for (int x = 0; x < d; ++x) gg += gu[x] * gu[x];
      for (int l = 0; l < T->W.n_loc; ++l) w[T->W.cell_dofs[K * T->W.n_loc + l]] = 1.0 / std::sqrt(1.0 + gg);
    }
    return 0;
  }
  if (kind == OK_GRADPOW_P0) {
    // W = P0, or QUAD (∇u_h of P1 is the same at every quadrature point of the cell)
    if ((T->W.family != OF_P0 && T->W.family != OF_QUAD) || T->V.family != OF_P1) return -2;
#pragma omp parallel for schedule(static)
    for (int64_t K = c0; K < c1; ++K) {
      Geo g = geometry(*T, K);
      const int32_t* I = &T->V.cell_dofs[K * T->V.n_loc];
      double gu[3] = {0, 0, 0};  // (Π_∇u ·₂ u) at the cell's DOF
      for (int a = 0; a <= d; ++a)
        for (int x = 0; x < d; ++x) gu[x] += u[I[a]] * g.grad[a][x];
      double nrm = 0;
      for (int x = 0; x < d; ++x) nrm += gu[x] * gu[x];
      nrm = std::sqrt(nrm);
      for (int l = 0; l < T->W.n_loc; ++l) w[T->W.cell_dofs[K * T->W.n_loc + l]] = std::pow(nrm, p - 2.0);
    }
    return 0;
  }
  if (kind == OK_P1_TO_P2_SQUARE) {
    if (T->W.family != OF_P2 || T->V.family != OF_P1 || d != 2) return -2;
    // DOF bary points of P2 local order v0,v1,v2,m01,m12,m20
    const double beta[6][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {0.5, 0.5, 0}, {0, 0.5, 0.5}, {0.5, 0, 0.5}};
    for (int64_t K = c0; K < c1; ++K) {
      const int32_t* I = &T->V.cell_dofs[K * 3];
      const int32_t* Wd = &T->W.cell_dofs[K * 6];
      for (int l = 0; l < 6; ++l) {
        double v = 0;  // (Π_u u)_k = Σ_j φ_j(x_k) u_j
        for (int a = 0; a < 3; ++a) v += beta[l][a] * u[I[a]];
        w[Wd[l]] = v * v;
      }
    }
    return 0;
  }
  return -3;
}

int oracle_interp(const void* h, int kind, double p, const double* u, double* w) {
  return oracle_interp_range(h, kind, p, u, w, 0, -1);
}

void oracle_set_threads(int n) { omp_set_num_threads(n < 1 ? 1 : n); }

// ---------------------------------------------------------------- apply
// r_i = Σ_{(j,k)} T_ijk u_j w_k, sequential in canonical order.
void oracle_apply(const void* h, const double* u, const double* w, double* r) {
  const OTensor* T = static_cast<const OTensor*>(h);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < T->V.n_dofs; ++i) {
    double acc = 0;
    for (int64_t e = T->t_row_ptr[i]; e < T->t_row_ptr[i + 1]; ++e)
      acc += T->t_val[e] * u[T->t_j[e]] * w[T->t_k[e]];
    r[i] = acc;
  }
}

// Batched: U, W, R pair-major (U[p*N_u + j], W[p*N_f + k], R[p*N_u + i]).
void oracle_apply_batched(const void* h, int32_t batch, const double* U, const double* W, double* R) {
  const OTensor* T = static_cast<const OTensor*>(h);
  for (int32_t p = 0; p < batch; ++p)
    oracle_apply(h, U + (int64_t)p * T->V.n_dofs, W + (int64_t)p * T->W.n_dofs, R + (int64_t)p * T->V.n_dofs);
}

// ---------------------------------------------------------------- jacobian
// D_u w as a list of (k, m, value) entries (pointwise Jacobian of the
// interpolated nonlinearity, "defined point-wise").
struct DEntry { int64_t k; int32_t m; double v; };

static int build_Duw(const OTensor* T, int kind, double p, const double* u, std::vector<DEntry>& D) {
  const int d = T->dim;
  if (T->W.family == OF_QUAD && (kind == OK_SQUARE || kind == OK_RECIPROCAL)) {
    // w_ℓ = f(u_h(x_ℓ)), u_h(x_ℓ) = Σ_a λ_a(x_ℓ) u_a  ⇒  ∂w_ℓ/∂u_a = f'(u_h(x_ℓ)) λ_a(x_ℓ)
    const int nq = T->W.n_loc;
    D.resize((size_t)T->n_cells * nq * (d + 1));  // entry order: cell, point, vertex (as a sequential push)
#pragma omp parallel for schedule(static)
    for (int64_t K = 0; K < T->n_cells; ++K) {
      const int32_t* I = &T->V.cell_dofs[K * T->V.n_loc];
      for (int l = 0; l < nq; ++l) {
        double uh = 0;
        for (int a = 0; a <= d; ++a) uh += T->wbary[l * (d + 1) + a] * u[I[a]];
        const double df = (kind == OK_SQUARE) ? 2.0 * uh : -1.0 / ((p + uh) * (p + uh));
        for (int a = 0; a <= d; ++a)
          D[((size_t)K * nq + l) * (d + 1) + a] = {(int64_t)T->W.cell_dofs[K * nq + l], I[a],
                                                    df * T->wbary[l * (d + 1) + a]};
      }
    }
    return 0;
  }
  if (kind == OK_IDENTITY) {
    for (int64_t k = 0; k < T->W.n_dofs; ++k) D.push_back({k, (int32_t)k, 1.0});
    return 0;
  }
  if (kind == OK_SQUARE) {
    for (int64_t k = 0; k < T->W.n_dofs; ++k) D.push_back({k, (int32_t)k, 2.0 * u[k]});
    return 0;
  }
  if (kind == OK_GRADPOW_P0) {
    // w_K = |g|^{p-2}, g = Σ_a u_a ∇λ_a  ⇒  ∂w_K/∂u_a = (p-2)|g|^{p-4} (g·∇λ_a);
    // at g = 0 the value 0 is used (reading C11).  W = QUAD: the same for every point of K.
    const int nl = T->W.n_loc;
    D.resize((size_t)T->n_cells * nl * (d + 1));  // entry order: cell, W-DOF, vertex (as a sequential push)
#pragma omp parallel for schedule(static)
    for (int64_t K = 0; K < T->n_cells; ++K) {
      Geo g = geometry(*T, K);
      const int32_t* I = &T->V.cell_dofs[K * T->V.n_loc];
      double gu[3] = {0, 0, 0};
      for (int a = 0; a <= d; ++a)
        for (int x = 0; x < d; ++x) gu[x] += u[I[a]] * g.grad[a][x];
      double gg = 0;
      for (int x = 0; x < d; ++x) gg += gu[x] * gu[x];
      double fac = (gg == 0.0) ? 0.0 : (p - 2.0) * std::pow(std::sqrt(gg), p - 4.0);
      for (int l = 0; l < nl; ++l)
        for (int a = 0; a <= d; ++a) {
          double gdot = 0;
          for (int x = 0; x < d; ++x) gdot += gu[x] * g.grad[a][x];
          D[((size_t)K * nl + l) * (d + 1) + a] = {(int64_t)T->W.cell_dofs[K * nl + l], I[a], fac * gdot};
        }
    }
    return 0;
  }
  if (kind == OK_MINSURF_P0) {
    // a_K = (1 + |g|²)^{-1/2}, g = Σ_a u_a ∇λ_a  ⇒  ∂a_K/∂u_a = −(1 + |g|²)^{-3/2} (g·∇λ_a)
    const int nl = T->W.n_loc;
    D.resize((size_t)T->n_cells * nl * (d + 1));
#pragma omp parallel for schedule(static)
    for (int64_t K = 0; K < T->n_cells; ++K) {
      Geo g = geometry(*T, K);
      const int32_t* I = &T->V.cell_dofs[K * T->V.n_loc];
      double gu[3] = {0, 0, 0};
      for (int a = 0; a <= d; ++a)
        for (int x = 0; x < d; ++x) gu[x] += u[I[a]] * g.grad[a][x];
      double gg = 0;
      for (int x = 0; x < d; ++x) gg += gu[x] * gu[x];
      const double fac = -std::pow(1.0 + gg, -1.5);
      for (int l = 0; l < nl; ++l)
        for (int a = 0; a <= d; ++a) {
          double gdot = 0;
          for (int x = 0; x < d; ++x) gdot += gu[x] * g.grad[a][x];
          D[((size_t)K * nl + l) * (d + 1) + a] = {(int64_t)T->W.cell_dofs[K * nl + l], I[a], fac * gdot};
        }
    }
    return 0;
  }
  if (kind == OK_RECIPROCAL) {
    // c̃ = 1/(k + u_h(x))  ⇒  ∂c̃/∂u_a = −λ_a(x)/(k + u_h(x))²  (x the W-DOF; λ_a = δ at nodes, 1/(d+1) at centroids)
    if (T->W.family == T->V.family && T->W.n_dofs == T->V.n_dofs) {
      for (int64_t k = 0; k < T->W.n_dofs; ++k) D.push_back({k, (int32_t)k, -1.0 / ((p + u[k]) * (p + u[k]))});
      return 0;
    }
    for (int64_t K = 0; K < T->n_cells; ++K) {
      const int32_t* I = &T->V.cell_dofs[K * T->V.n_loc];
      double uc = 0;
      for (int a = 0; a <= d; ++a) uc += u[I[a]] / (d + 1);
      for (int a = 0; a <= d; ++a)
        D.push_back({(int64_t)T->W.cell_dofs[K], I[a], -1.0 / ((d + 1) * (p + uc) * (p + uc))});
    }
    return 0;
  }
  if (kind == OK_P1_TO_P2_SQUARE) {
    // w = (Π u)⊙(Π u) ⇒ D = diag(2 Π u) Π; only the nonzero entries of Π.
    const double beta[6][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {0.5, 0.5, 0}, {0, 0.5, 0.5}, {0.5, 0, 0.5}};
    std::map<std::pair<int64_t, int32_t>, double> Dm;
    for (int64_t K = 0; K < T->n_cells; ++K) {
      const int32_t* I = &T->V.cell_dofs[K * 3];
      const int32_t* Wd = &T->W.cell_dofs[K * 6];
      for (int l = 0; l < 6; ++l) {
        double v = 0;
        for (int a = 0; a < 3; ++a) v += beta[l][a] * u[I[a]];
        for (int a = 0; a < 3; ++a)
          if (beta[l][a] != 0.0) Dm[{(int64_t)Wd[l], I[a]}] = 2.0 * v * beta[l][a];
      }
    }
    for (auto& kv : Dm) D.push_back({kv.first.first, kv.first.second, kv.second});
    return 0;
  }
  return -1;
}

// ---------------------------------------------------------------- bilinear GFEM form (F3)
// B_ik = ∫ (opA φ_i)(opC η_k): the matrix of PAPER.md L196–203 (M^c: MASS3's slots) and
// L402–409 (N^f: CONV_I's), assembled element by element with its own quadrature (degree of
// the bilinear integrand), into the CSR pattern (W = V numbering).  Independent of T.
int oracle_bilinear(const void* h, double* vals) {
  const OTensor* T = static_cast<const OTensor*>(h);
  const int d = T->dim;
  if (T->W.n_dofs != T->V.n_dofs || T->W.family != T->V.family) return -1;
  int opA, opB, opC;
  form_ops(T->form, &opA, &opB, &opC);
  (void)opB;
  if (opA == OP_GRAD) return -2;  // ∫ η ∇φ_i is a vector: no scalar bilinear form
  Rule R = default_rule(d, op_degree(opA, T->V.family) + op_degree(opC, T->W.family));
  std::fill(vals, vals + T->csr_col.size(), 0.0);
  const int nA = T->V.n_loc, nC = T->W.n_loc;
  std::vector<double> vv(nA), wv(nC), vg(nA * 3), wg(nC * 3);
  for (int64_t K = 0; K < T->n_cells; ++K) {
    Geo g = geometry(*T, K);
    const int32_t* I = &T->V.cell_dofs[K * nA];
    const int32_t* Wd = &T->W.cell_dofs[K * nC];
    for (int q = 0; q < R.nq; ++q) {
      const double* lam = &R.bary[q * (d + 1)];
      basis(T->V.family, d, lam, g, nA, vv.data(), reinterpret_cast<double(*)[3]>(vg.data()));
      basis(T->W.family, d, lam, g, nC, wv.data(), reinterpret_cast<double(*)[3]>(wg.data()));
      const double wq = R.w[q] * g.vol;
      for (int a = 0; a < nA; ++a) {
        if (I[a] < T->row_begin || I[a] >= T->row_end) continue;
        for (int c = 0; c < nC; ++c) {
          const int64_t sl = csr_find(T, I[a], Wd[c]);
          if (sl < 0) return -3;
          vals[sl] += wq * apply_op(opA, d, vv[a], &vg[a * 3]) * apply_op(opC, d, wv[c], &wg[c * 3]);
        }
      }
    }
  }
  return 0;
}

// csr_vals = T·w                                    (PICARD)
// csr_vals = T·w + (T·₂u)·D_u w                     (NEWTON)
int oracle_jacobian(const void* h, int mode, int kind, double p, const double* u, const double* w,
                    double* vals) {
  const OTensor* T = static_cast<const OTensor*>(h);
  std::fill(vals, vals + T->csr_col.size(), 0.0);
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(|| : bad)
  for (int64_t i = 0; i < T->V.n_dofs; ++i)
    for (int64_t e = T->t_row_ptr[i]; e < T->t_row_ptr[i + 1]; ++e) {
      int64_t s = csr_find(T, i, T->t_j[e]);
      if (s < 0) {
        bad = 1;
        break;
      }
      vals[s] += T->t_val[e] * w[T->t_k[e]];
    }
  if (bad) return -3;
  if (mode == OJ_PICARD) return 0;
  std::vector<DEntry> D;
  int rc = build_Duw(T, kind, p, u, D);
  if (rc) return rc;
  // index D by k (stable: entries of one k keep insertion order)
  std::vector<int64_t> dptr(T->W.n_dofs + 1, 0);
  for (auto& de : D) dptr[de.k + 1]++;
  for (int64_t k = 0; k < T->W.n_dofs; ++k) dptr[k + 1] += dptr[k];
  std::vector<DEntry> Ds(D.size());
  {
    std::vector<int64_t> fill(dptr.begin(), dptr.end() - 1);
    for (auto& de : D) Ds[fill[de.k]++] = de;
  }
#pragma omp parallel for schedule(static) reduction(|| : bad)
  for (int64_t i = 0; i < T->V.n_dofs; ++i) {
    // B_{i,k} = (T ·₂ u)_{ik} = Σ_j T_ijk u_j
    std::map<int64_t, double> B;
    for (int64_t e = T->t_row_ptr[i]; e < T->t_row_ptr[i + 1]; ++e)
      B[T->t_k[e]] += T->t_val[e] * u[T->t_j[e]];
    for (auto& kv : B)
      for (int64_t q = dptr[kv.first]; q < dptr[kv.first + 1]; ++q) {
        int64_t s = csr_find(T, i, Ds[q].m);
        if (s < 0) {
          bad = 1;
          continue;
        }
        vals[s] += kv.second * Ds[q].v;
      }
  }
  return bad ? -6 : 0;
}

}  // extern "C"

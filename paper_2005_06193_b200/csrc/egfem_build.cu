// Offline tensor builder of libegfem.so (PAPER.md L196–203 eq.
// (egfem_terms), L304 "offline phase").
//
//   1. one thread per cell computes the local tensor T_K[a][b][c] by quadrature
//      (geometry by cross products, Lagrange P0/P1/P2 bases in barycentric
//      coordinates) and emits every structural triple (I[a], J[b], W[c], value);
//   2. a stable CUB radix sort orders the triples lexicographically by (i, j, k):
//      one pass on the packed key when it fits 64 bits, otherwise an LSD pair of
//      passes (k, then (i,j)) — the (i,j,k) key overflows 64 bits for cfg4;
//   3. duplicates are summed in emission order, fibers (i,j) and rows are
//      delimited by flag/scan, P0 local indices are packed into nz_k, and rows are
//      grouped into shared-memory tiles.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "egfem_internal.cuh"
#include "egfem_interp.cuh"

namespace egfem {
namespace {

enum SlotOp { kValue = 0, kDx = 1, kDxDy = 2, kGrad = 3 };

struct ElemParams {
  int dim, nV, nW, vfam, wfam;
  int opA, opB, opC;
  int nq;
  double bary[kMaxQuad * 4];
  double wq[kMaxQuad];
  int64_t n_cells, n_u;
  const double* coords;
  const int32_t* cells;
  const int32_t* vdofs;
  const int32_t* wdofs;
  uint64_t* key;
  uint32_t* kout;
  double* val;
};

// Gradients of the barycentric coordinates of a simplex and its measure.
// 3D: ∇λ_a = (e_b × e_c)/det for the cyclic (a,b,c) of edges e_a = x_a − x_0;
// 2D: ∇λ_1 = (e2y, −e2x)/det, ∇λ_2 = (−e1y, e1x)/det;  ∇λ_0 = −Σ_{a≥1} ∇λ_a.
__device__ __forceinline__ double simplex_gradients(int d, const double (*x)[3], double (*g)[3]) {
  double vol;
  for (int a = 0; a < 4; ++a) g[a][0] = g[a][1] = g[a][2] = 0.0;
  if (d == 1) {
    double h = x[1][0] - x[0][0];
    g[1][0] = 1.0 / h;
    vol = fabs(h);
  } else if (d == 2) {
    double e1x = x[1][0] - x[0][0], e1y = x[1][1] - x[0][1];
    double e2x = x[2][0] - x[0][0], e2y = x[2][1] - x[0][1];
    double det = e1x * e2y - e1y * e2x;
    g[1][0] = e2y / det;
    g[1][1] = -e2x / det;
    g[2][0] = -e1y / det;
    g[2][1] = e1x / det;
    vol = 0.5 * fabs(det);
  } else {
    double e[3][3];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) e[a][c] = x[a + 1][c] - x[0][c];
    double c23[3] = {e[1][1] * e[2][2] - e[1][2] * e[2][1], e[1][2] * e[2][0] - e[1][0] * e[2][2],
                     e[1][0] * e[2][1] - e[1][1] * e[2][0]};
    double c31[3] = {e[2][1] * e[0][2] - e[2][2] * e[0][1], e[2][2] * e[0][0] - e[2][0] * e[0][2],
                     e[2][0] * e[0][1] - e[2][1] * e[0][0]};
    double c12[3] = {e[0][1] * e[1][2] - e[0][2] * e[1][1], e[0][2] * e[1][0] - e[0][0] * e[1][2],
                     e[0][0] * e[1][1] - e[0][1] * e[1][0]};
    double det = e[0][0] * c23[0] + e[0][1] * c23[1] + e[0][2] * c23[2];
    for (int c = 0; c < 3; ++c) {
      g[1][c] = c23[c] / det;
      g[2][c] = c31[c] / det;
      g[3][c] = c12[c] / det;
    }
    vol = fabs(det) / 6.0;
  }
  for (int c = 0; c < d; ++c) {
    double s = 0.0;
    for (int a = 1; a <= d; ++a) s += g[a][c];
    g[0][c] = -s;
  }
  return vol;
}

// Local Lagrange basis at barycentric point lam: values and physical gradients.
// P2 (2D): vertex a: λ_a(2λ_a − 1); edge (a,b) in order m01, m12, m20: 4λ_aλ_b.
__device__ __forceinline__ void eval_basis(int fam, int d, const double* lam, const double (*g)[3], double* v,
                                           double (*gr)[3]) {
  if (fam == EGFEM_P0) {
    v[0] = 1.0;
    gr[0][0] = gr[0][1] = gr[0][2] = 0.0;
  } else if (fam == EGFEM_P1) {
    for (int a = 0; a <= d; ++a) {
      v[a] = lam[a];
      for (int c = 0; c < 3; ++c) gr[a][c] = g[a][c];
    }
  } else {
    for (int a = 0; a < 3; ++a) {
      v[a] = lam[a] * (2.0 * lam[a] - 1.0);
      for (int c = 0; c < 3; ++c) gr[a][c] = (4.0 * lam[a] - 1.0) * g[a][c];
    }
    const int ea[3] = {0, 1, 2}, eb[3] = {1, 2, 0};
    for (int m = 0; m < 3; ++m) {
      int a = ea[m], b = eb[m];
      v[3 + m] = 4.0 * lam[a] * lam[b];
      for (int c = 0; c < 3; ++c) gr[3 + m][c] = 4.0 * (lam[a] * g[b][c] + lam[b] * g[a][c]);
    }
  }
}

__device__ __forceinline__ double slot_value(int op, int d, double v, const double* gr) {
  switch (op) {
    case kValue: return v;
    case kDx: return gr[0];
    default: return d >= 2 ? gr[0] + gr[1] : gr[0];  // (∂x + ∂y)
  }
}

__global__ void k_element_triples(const ElemParams P) {
  int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= P.n_cells) return;
  const int d = P.dim, nV = P.nV, nW = P.nW, L = nV * nV * nW;
  double x[4][3] = {{0}};
  for (int a = 0; a <= d; ++a) {
    int64_t v = P.cells[cell * (d + 1) + a];
    for (int c = 0; c < d; ++c) x[a][c] = P.coords[v * d + c];
  }
  double g[4][3];
  double vol = simplex_gradients(d, x, g);
  double Tl[256];
  for (int l = 0; l < L; ++l) Tl[l] = 0.0;
  double fv[6], gv[6][3], fw[kMaxQuad], gw[kMaxQuad][3];
  for (int q = 0; q < P.nq; ++q) {
    const double* lam = &P.bary[q * (d + 1)];
    eval_basis(P.vfam, d, lam, g, fv, gv);
    if (P.wfam == EGFEM_QUAD) {  // η_ℓ = w_ℓ δ_{x_ℓ}: the ℓ-th DOF "evaluates" to δ_{ℓq}
      for (int c = 0; c < nW; ++c) {
        fw[c] = (c == q) ? 1.0 : 0.0;
        gw[c][0] = gw[c][1] = gw[c][2] = 0.0;
      }
    } else {
      eval_basis(P.wfam, d, lam, g, fw, gw);
    }
    const double wq = P.wq[q] * vol;
    for (int a = 0; a < nV; ++a)
      for (int b = 0; b < nV; ++b) {
        double fab;
        if (P.opA == kGrad) {
          fab = 0.0;
          for (int c = 0; c < d; ++c) fab += gv[a][c] * gv[b][c];
        } else {
          fab = slot_value(P.opA, d, fv[a], gv[a]) * slot_value(P.opB, d, fv[b], gv[b]);
        }
        for (int c = 0; c < nW; ++c) Tl[(a * nV + b) * nW + c] += wq * fab * slot_value(P.opC, d, fw[c], gw[c]);
      }
  }
  const int64_t base = cell * L;
  for (int a = 0; a < nV; ++a) {
    uint64_t i = (uint64_t)P.vdofs[cell * nV + a];
    for (int b = 0; b < nV; ++b) {
      uint64_t j = (uint64_t)P.vdofs[cell * nV + b];
      for (int c = 0; c < nW; ++c) {
        int64_t o = base + (a * nV + b) * nW + c;
        P.key[o] = i * (uint64_t)P.n_u + j;
        P.kout[o] = (uint32_t)P.wdofs[cell * nW + c];
        P.val[o] = Tl[(a * nV + b) * nW + c];
      }
    }
  }
}

// (cc, inv3) of each geometry class from its edge vectors, by the interp's own cof3 (bitwise the
// per-cell evaluation): e is 9 x nk (class-major), gtab 10 x nk (value-major)
__global__ void k_geo_table(const double* e, int nk, double* gtab) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nk) return;
  double ee[3][3], cc[3][3], inv3;
  for (int a = 0; a < 3; ++a)
    for (int q = 0; q < 3; ++q) ee[a][q] = e[k * 9 + a * 3 + q];
  ip::cof3(ee, cc, inv3);
  for (int a = 0; a < 3; ++a)
    for (int q = 0; q < 3; ++q) gtab[(a * 3 + q) * nk + k] = cc[a][q];
  gtab[9 * nk + k] = inv3;
}

__global__ void k_iota(uint32_t* a, int64_t n) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) a[e] = (uint32_t)e;
}

__global__ void k_pack_key(const uint64_t* kij, const uint32_t* k, int kbits, uint64_t* out, int64_t n) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) out[e] = (kij[e] << kbits) | (uint64_t)k[e];
}

template <typename T>
__global__ void k_gather(const T* src, const uint32_t* idx, T* dst, int64_t n) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = src[idx[e]];
}

__global__ void k_unique_flags(const uint64_t* key, const uint32_t* k, int32_t* flag, int64_t n) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) flag[e] = (e == 0 || key[e] != key[e - 1] || k[e] != k[e - 1]) ? 1 : 0;
}

__global__ void k_mark_starts(const int32_t* flag, const int64_t* pos, int64_t* start, int64_t n) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n && flag[e]) start[pos[e]] = e;
}

// Sum each duplicate run sequentially in emission order (stable sort keeps it).
__global__ void k_reduce_runs(const int64_t* start, int64_t nu, int64_t m, const uint64_t* key, const uint32_t* k,
                              const double* val, uint64_t* okey, uint32_t* ok, double* oval) {
  int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nu) return;
  int64_t s = start[u], e = (u + 1 < nu) ? start[u + 1] : m;
  double acc = 0.0;
  for (int64_t x = s; x < e; ++x) acc += val[x];
  okey[u] = key[s];
  ok[u] = k[s];
  oval[u] = acc;
}

__global__ void k_fiber_flags(const uint64_t* key, int32_t* flag, int64_t n) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) flag[e] = (e == 0 || key[e] != key[e - 1]) ? 1 : 0;
}

__global__ void k_fiber_fill(const int32_t* flag, const int64_t* pos, const uint64_t* key, int64_t n_u, int64_t nnz,
                             uint32_t* fib_nz, int32_t* fib_j, int64_t* row_cnt) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz || !flag[e]) return;
  int64_t f = pos[e];
  fib_nz[f] = (uint32_t)e;
  fib_j[f] = (int32_t)(key[e] % (uint64_t)n_u);
  atomicAdd((unsigned long long*)&row_cnt[key[e] / (uint64_t)n_u], 1ull);  // integer: deterministic
}

__global__ void k_pack_loc(const uint64_t* key, uint32_t* nz_k, int64_t nnz, int64_t n_u, const int32_t* wcell,
                           const int32_t* vdofs, int nV, int* err) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  int32_t j = (int32_t)(key[e] % (uint64_t)n_u);
  uint32_t K = nz_k[e];
  int64_t c = wcell[K];
  int m = -1;
  for (int a = 0; a < nV; ++a)
    if (vdofs[c * nV + a] == j) m = a;
  if (m < 0 || m > 3) {
    atomicExch(err, 1);
    return;
  }
  nz_k[e] = K | ((uint32_t)m << kKShift);
}

// slot = number of cells of row i (k's of the diagonal fiber (i,i)) below k; requires
// slot*(d+1)+loc_j < row nnz, i.e. every row is (d+1) x (cells around i) — true for P1 V.
__global__ void k_cell_slot(const uint64_t* key, int64_t nnz, int64_t n_u, const int64_t* row_fib,
                            const int32_t* fib_j, const uint32_t* fib_nz, const uint32_t* nz_k, int nV,
                            uint8_t* aux, int* err) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  const int64_t i = (int64_t)(key[e] / (uint64_t)n_u);
  int64_t lo = row_fib[i], hi = row_fib[i + 1];
  const int64_t f_end = hi;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (fib_j[mid] < (int32_t)i) lo = mid + 1; else hi = mid;
  }
  if (lo >= f_end || fib_j[lo] != (int32_t)i) {
    atomicExch(err, 1);
    return;
  }
  const uint32_t K = nz_k[e] & kKMask;
  uint32_t a = fib_nz[lo], b = fib_nz[lo + 1];
  const uint32_t d0 = a;
  while (a < b) {
    uint32_t mid = (a + b) / 2;
    if ((nz_k[mid] & kKMask) < K) a = mid + 1; else b = mid;
  }
  const int64_t slot = (int64_t)a - d0;
  const int64_t row_nnz = (int64_t)fib_nz[row_fib[i + 1]] - (int64_t)fib_nz[row_fib[i]];
  const int m = (int)((nz_k[e] >> kKShift) & 3u);
  if (slot > 255 || slot * nV + m >= row_nnz || a >= fib_nz[lo + 1] || (nz_k[a] & kKMask) != K) {
    atomicExch(err, 1);
    return;
  }
  aux[e] = (uint8_t)slot;
}

__global__ void k_heads(const uint32_t* fib_nz, int64_t n_fib, uint32_t* nz_k) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f < n_fib && fib_nz[f] < fib_nz[f + 1]) nz_k[fib_nz[f]] |= kHead;
}

__global__ void k_row_nz(const int64_t* row_fib, const uint32_t* fib_nz, int64_t n_u, int64_t* row_nz) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n_u) row_nz[i] = fib_nz[row_fib[i]];
}

__global__ void k_to_f32(const double* a, float* b, int64_t n) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) b[e] = (float)a[e];
}

__global__ void k_wcell(const int32_t* wdofs, int nw, int32_t* wcell, int64_t n_cells) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n_cells)
    for (int l = 0; l < nw; ++l) wcell[wdofs[c * nw + l]] = (int32_t)c;
}

inline int nblk(int64_t n, int t = 256) { return (int)((n + t - 1) / t); }

inline int bits_for(uint64_t maxval) {
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

// RAII device buffer for builder temporaries.
template <typename T>
struct DBuf {
  T* p = nullptr;
  cudaError_t alloc(int64_t n) { return cudaMalloc(&p, sizeof(T) * (size_t)std::max<int64_t>(n, 1)); }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  T* release() {
    T* q = p;
    p = nullptr;
    return q;
  }
};

// Default quadrature rules (weights sum to 1; readings C2/C3).
void default_rule(int d, int degree, int* nq, double* bary, double* wq) {
  if (d == 1) {
    const double s = std::sqrt(0.6);
    const double xi[3] = {0.5 - 0.5 * s, 0.5, 0.5 + 0.5 * s};
    const double w[3] = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};
    *nq = 3;
    for (int q = 0; q < 3; ++q) {
      bary[2 * q] = 1.0 - xi[q];
      bary[2 * q + 1] = xi[q];
      wq[q] = w[q];
    }
  } else if (d == 2 && degree <= 1) {
    *nq = 1;
    bary[0] = bary[1] = bary[2] = 1.0 / 3.0;
    wq[0] = 1.0;
  } else if (d == 2 && degree == 2) {
    *nq = 3;
    for (int q = 0; q < 3; ++q) {
      for (int a = 0; a < 3; ++a) bary[3 * q + a] = (a == q) ? 2.0 / 3.0 : 1.0 / 6.0;
      wq[q] = 1.0 / 3.0;
    }
  } else if (d == 2) {
    // Symmetric 6-point rule, degree 4 (Dunavant): orbits (1−2a, a, a).
    const double orbit_a[2] = {0.445948490915965, 0.091576213509770549};
    const double orbit_w[2] = {0.2233815896780118, 0.10995174365532154};
    *nq = 6;
    for (int o = 0; o < 2; ++o)
      for (int q = 0; q < 3; ++q) {
        for (int a = 0; a < 3; ++a) bary[3 * (3 * o + q) + a] = (a == q) ? 1.0 - 2.0 * orbit_a[o] : orbit_a[o];
        wq[3 * o + q] = orbit_w[o];
      }
  } else if (degree <= 1) {
    *nq = 1;
    for (int a = 0; a < 4; ++a) bary[a] = 0.25;
    wq[0] = 1.0;
  } else if (degree >= 3) {
    // Symmetric 14-point rule, degree 5, positive weights: two S31 orbits (1−3a, a, a, a) and
    // one S22 orbit (c, c, ½−c, ½−c).  Constants solved from the |α| ≤ 5 moment equations in
    // 50-digit arithmetic (scripts/tet14_rule.py); exact for every 3D P1 form (MASS3 is degree 3,
    // PAPER.md L327).  Callers never ask for degree > 5 in 3D (P2 is 2D only).
    const double orbit_a[2] = {0.092735250310891226, 0.31088591926330061};
    const double orbit_w[2] = {0.07349304311636195, 0.11268792571801585};
    const double c = 0.045503704125649649, wc = 0.042546020777081466;
    *nq = 14;
    int q = 0;
    for (int o = 0; o < 2; ++o)
      for (int v = 0; v < 4; ++v, ++q) {
        for (int a = 0; a < 4; ++a) bary[4 * q + a] = (a == v) ? 1.0 - 3.0 * orbit_a[o] : orbit_a[o];
        wq[q] = orbit_w[o];
      }
    for (int x = 0; x < 4; ++x)
      for (int y = x + 1; y < 4; ++y, ++q) {
        for (int a = 0; a < 4; ++a) bary[4 * q + a] = (a == x || a == y) ? c : 0.5 - c;
        wq[q] = wc;
      }
  } else {
    const double a = 0.1381966011250105, b = 0.5854101966249685;
    *nq = 4;
    for (int q = 0; q < 4; ++q) {
      for (int c = 0; c < 4; ++c) bary[4 * q + c] = (c == q) ? b : a;
      wq[q] = 0.25;
    }
  }
}

// The default rule with exactly n points (QUAD W without an explicit rule); false if none.
bool default_rule_points(int d, int n, int* nq, double* bary, double* wq) {
  const int deg = d == 1 ? (n == 3 ? 5 : -1)
                  : d == 2 ? (n == 1 ? 1 : n == 3 ? 2 : n == 6 ? 4 : -1)
                           : (n == 1 ? 1 : n == 4 ? 2 : -1);
  if (deg < 0) return false;
  default_rule(d, deg, nq, bary, wq);
  return *nq == n;
}

int fam_degree(int f) { return (f == EGFEM_P0 || f == EGFEM_QUAD) ? 0 : (f == EGFEM_P1 ? 1 : 2); }
int op_degree(int op, int fam) {
  int p = fam_degree(fam);
  return op == kValue ? p : (p > 0 ? p - 1 : 0);
}

}  // namespace

egfem_status upload_mesh(egfem_tensor* t, const egfem_mesh* mesh, const egfem_space* V, const egfem_space* W) {
  const int d = mesh->dim;
  t->has_mesh = true;
  t->dim = d;
  t->n_vertices = mesh->n_vertices;
  t->n_cells = mesh->n_cells;
  t->vfam = V->family;
  t->wfam = W->family;
  const int64_t nq = W->family == EGFEM_QUAD ? W->n_dofs / mesh->n_cells : 0;
  auto nloc = [d, nq](egfem_family f) {
    return f == EGFEM_P0 ? 1 : f == EGFEM_P1 ? d + 1 : f == EGFEM_QUAD ? (int)nq : 6;
  };
  t->nV = nloc(V->family);
  t->nW = nloc(W->family);
  t->n_u = V->n_dofs;
  t->n_f = W->n_dofs;
  const int64_t nc = mesh->n_cells;
  std::vector<int32_t> tmp;
  auto table = [&](const egfem_space* S, int nl) -> const int32_t* {
    if (S->cell_dofs) return S->cell_dofs;
    tmp.resize((size_t)nc * nl);
    for (int64_t c = 0; c < nc; ++c)
      for (int a = 0; a < nl; ++a)
        tmp[c * nl + a] = S->family == EGFEM_P0     ? (int32_t)c
                          : S->family == EGFEM_QUAD ? (int32_t)(c * nl + a)
                                                    : mesh->cells[c * (d + 1) + a];
    return tmp.data();
  };
  EGFEM_CUDA_TRY(cudaMalloc(&t->coords, sizeof(double) * mesh->n_vertices * d));
  EGFEM_CUDA_TRY(cudaMemcpy(t->coords, mesh->coords, sizeof(double) * mesh->n_vertices * d, cudaMemcpyHostToDevice));
  EGFEM_CUDA_TRY(cudaMalloc(&t->cells, sizeof(int32_t) * nc * (d + 1)));
  EGFEM_CUDA_TRY(cudaMemcpy(t->cells, mesh->cells, sizeof(int32_t) * nc * (d + 1), cudaMemcpyHostToDevice));
  const int32_t* hv = table(V, t->nV);
  EGFEM_CUDA_TRY(cudaMalloc(&t->vdofs, sizeof(int32_t) * nc * t->nV));
  EGFEM_CUDA_TRY(cudaMemcpy(t->vdofs, hv, sizeof(int32_t) * nc * t->nV, cudaMemcpyHostToDevice));
  std::vector<int32_t> hvcopy(hv, hv + (size_t)nc * t->nV);
  const int32_t* hw = table(W, t->nW);
  EGFEM_CUDA_TRY(cudaMalloc(&t->wdofs, sizeof(int32_t) * nc * t->nW));
  EGFEM_CUDA_TRY(cudaMemcpy(t->wdofs, hw, sizeof(int32_t) * nc * t->nW, cudaMemcpyHostToDevice));
  t->vdofs_is_cells = (V->family == EGFEM_P1) && std::equal(hvcopy.begin(), hvcopy.end(), mesh->cells);
  if (W->family == EGFEM_P0 || W->family == EGFEM_QUAD) {  // canonical cell-wise numbering: (c, l) -> c·nW + l
    t->wdofs_is_iota = true;
    for (int64_t x = 0; x < nc * t->nW && t->wdofs_is_iota; ++x) t->wdofs_is_iota = (hw[x] == (int32_t)x);
  }
  if (d == 3) {
    std::vector<double> c4((size_t)mesh->n_vertices * 4, 0.0);
    for (int64_t v = 0; v < mesh->n_vertices; ++v)
      for (int q = 0; q < 3; ++q) c4[v * 4 + q] = mesh->coords[v * 3 + q];
    EGFEM_CUDA_TRY(cudaMalloc(&t->coords4, sizeof(double) * c4.size()));
    EGFEM_CUDA_TRY(cudaMemcpy(t->coords4, c4.data(), sizeof(double) * c4.size(), cudaMemcpyHostToDevice));
    // lossless 16-byte copy when every coordinate is exactly representable as a float (e.g. the
    // structured meshes, coordinates i/n with n a power of two): half the gather bytes and registers
    bool exact = true;
    for (double x : c4)
      if ((double)(float)x != x) {
        exact = false;
        break;
      }
    if (exact) {
      std::vector<float> c4f(c4.begin(), c4.end());
      EGFEM_CUDA_TRY(cudaMalloc(&t->coordsf, sizeof(float) * c4f.size()));
      EGFEM_CUDA_TRY(cudaMemcpy(t->coordsf, c4f.data(), sizeof(float) * c4f.size(), cudaMemcpyHostToDevice));
    }
  }
  if (d == 2) {  // lossless float2 copy when every coordinate is exactly a float
    const int64_t nv2 = (int64_t)mesh->n_vertices * 2;
    bool exact = true;
    for (int64_t x = 0; x < nv2 && exact; ++x) exact = (double)(float)mesh->coords[x] == mesh->coords[x];
    if (exact) {
      std::vector<float> c2f(mesh->coords, mesh->coords + nv2);
      EGFEM_CUDA_TRY(cudaMalloc(&t->coordsf, sizeof(float) * std::max<int64_t>(nv2, 1)));
      EGFEM_CUDA_TRY(cudaMemcpy(t->coordsf, c2f.data(), sizeof(float) * nv2, cudaMemcpyHostToDevice));
    }
  }
  t->w_is_v = (V->family == W->family) && (V->n_dofs == W->n_dofs) &&
              std::equal(hvcopy.begin(), hvcopy.end(), hw);
  t->w_p0 = (W->family == EGFEM_P0 || W->family == EGFEM_QUAD);
  t->nwc = t->w_p0 ? t->nW : 1;
  t->newton_wv_ok = t->w_is_v;  // k and j of a cell share it: (i, k) is an element-clique pair
  if (t->w_p0) {
    EGFEM_CUDA_TRY(cudaMalloc(&t->wcell, sizeof(int32_t) * std::max<int64_t>(t->n_f, 1)));
    k_wcell<<<nblk(nc), 256>>>(t->wdofs, t->nW, t->wcell, nc);
    count_launch();
    EGFEM_CUDA_TRY(cudaGetLastError());
  }
  return make_geo_classes(t, mesh);
}

// Geometry classes for the 3D interp of the gradient kinds (canonical P1 V / P0 W): a cell's
// interp reads only u at its vertices and the (cc, inv3) of its class when every cell's edge
// vectors x_{a+1} − x_0 (exact double differences, as the kernel forms them) are bitwise one of at
// most kMaxGeoClasses tuples — meshes made of translated copies of a few cells (the structured
// meshes of the paper's experiments).  Otherwise (or EGFEM_GEOM_CLASSES=0) no table: the
// interp gathers the coordinates.
egfem_status make_geo_classes(egfem_tensor* t, const egfem_mesh* mesh) {
  if (t->dim != 3 || !t->vdofs_is_cells || !t->wdofs_is_iota || !t->w_p0 || t->nwc != 1) return EGFEM_OK;
  const char* env = std::getenv("EGFEM_GEOM_CLASSES");
  if (env && env[0] == '0') return EGFEM_OK;
  const int64_t nc = mesh->n_cells;
  std::vector<double> reps;  // 9 per class
  std::vector<uint8_t> cls((size_t)nc);
  int last = 0;
  for (int64_t c = 0; c < nc; ++c) {
    const int32_t* v = mesh->cells + c * 4;
    double e[9];
    for (int a = 0; a < 3; ++a)
      for (int q = 0; q < 3; ++q) e[a * 3 + q] = mesh->coords[(int64_t)v[a + 1] * 3 + q] - mesh->coords[(int64_t)v[0] * 3 + q];
    const int nk = (int)(reps.size() / 9);
    int k = -1;
    for (int i = 0; i < nk && k < 0; ++i) {
      const int cand = (last + i) % nk;  // the previous cell's class first
      if (std::memcmp(e, &reps[(size_t)cand * 9], sizeof(e)) == 0) k = cand;
    }
    if (k < 0) {
      if (nk == kMaxGeoClasses) return EGFEM_OK;  // not a few-class mesh: the gathering interp
      reps.insert(reps.end(), e, e + 9);
      k = nk;
    }
    cls[(size_t)c] = (uint8_t)k;
    last = k;
  }
  const int nk = (int)(reps.size() / 9);
  double* de = nullptr;
  EGFEM_CUDA_TRY(cudaMalloc(&de, sizeof(double) * reps.size()));
  EGFEM_CUDA_TRY(cudaMemcpy(de, reps.data(), sizeof(double) * reps.size(), cudaMemcpyHostToDevice));
  EGFEM_CUDA_TRY(cudaMalloc(&t->gtab, sizeof(double) * 10 * nk));
  k_geo_table<<<1, 64>>>(de, nk, t->gtab);
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  EGFEM_CUDA_TRY(cudaDeviceSynchronize());
  cudaFree(de);
  EGFEM_CUDA_TRY(cudaMalloc(&t->gcls, std::max<int64_t>(nc, 16)));
  EGFEM_CUDA_TRY(cudaMemcpy(t->gcls, cls.data(), nc, cudaMemcpyHostToDevice));
  t->n_geo = nk;
  return EGFEM_OK;
}

egfem_status emit_element_triples(egfem_tensor* t, egfem_form form, const egfem_quad* quad, int64_t* m_out,
                                  uint64_t** key, uint32_t** k, double** val) {
  ElemParams P{};
  P.dim = t->dim;
  P.nV = t->nV;
  P.nW = t->nW;
  P.vfam = t->vfam;
  P.wfam = t->wfam;
  switch (form) {
    case EGFEM_FORM_CONV_K: P.opA = kValue; P.opB = kValue; P.opC = kDx; break;
    case EGFEM_FORM_CONV_J: P.opA = kValue; P.opB = kDxDy; P.opC = kValue; break;
    case EGFEM_FORM_PLAP: P.opA = kGrad; P.opB = kGrad; P.opC = kValue; break;
    case EGFEM_FORM_MASS3: P.opA = kValue; P.opB = kValue; P.opC = kValue; break;
    default: P.opA = kDxDy; P.opB = kValue; P.opC = kValue; break;
  }
  if (quad && quad->n_points > 0) {
    if (quad->n_points > kMaxQuad) {
      set_error("quadrature with more than 16 points");
      return EGFEM_ERR_UNSUPPORTED;
    }
    P.nq = quad->n_points;
    for (int q = 0; q < P.nq; ++q) {
      for (int a = 0; a <= t->dim; ++a) P.bary[q * (t->dim + 1) + a] = quad->bary[q * (t->dim + 1) + a];
      P.wq[q] = quad->weights[q];
    }
  } else if (t->wfam == EGFEM_QUAD) {  // I_k: the default rule with N_q = nW points
    if (!default_rule_points(t->dim, t->nW, &P.nq, P.bary, P.wq)) {
      set_error("QUAD W: no default rule with " + std::to_string(t->nW) + " points in " + std::to_string(t->dim) +
                "D (pass egfem_quad)");
      return EGFEM_ERR_UNSUPPORTED;
    }
  } else {
    int deg = (P.opA == kGrad) ? 2 * op_degree(kDx, t->vfam) + op_degree(kValue, t->wfam)
                               : op_degree(P.opA, t->vfam) + op_degree(P.opB, t->vfam) + op_degree(P.opC, t->wfam);
    default_rule(t->dim, deg, &P.nq, P.bary, P.wq);
  }
  // cell-wise W: barycentric coordinates of each cell's W DOFs (P0: centroid; QUAD: the rule)
  if (t->w_p0) {
    std::vector<double> pts((size_t)t->nwc * (t->dim + 1));
    for (int l = 0; l < t->nwc; ++l)
      for (int a = 0; a <= t->dim; ++a)
        pts[l * (t->dim + 1) + a] = t->wfam == EGFEM_QUAD ? P.bary[l * (t->dim + 1) + a] : 1.0 / (t->dim + 1);
    EGFEM_CUDA_TRY(cudaMalloc(&t->wpts, sizeof(double) * pts.size()));
    EGFEM_CUDA_TRY(cudaMemcpy(t->wpts, pts.data(), sizeof(double) * pts.size(), cudaMemcpyHostToDevice));
  }
  P.n_cells = t->n_cells;
  P.n_u = t->n_u;
  P.coords = t->coords;
  P.cells = t->cells;
  P.vdofs = t->vdofs;
  P.wdofs = t->wdofs;
  const int64_t m = t->n_cells * (int64_t)t->nV * t->nV * t->nW;
  EGFEM_CUDA_TRY(cudaMalloc(key, sizeof(uint64_t) * std::max<int64_t>(m, 1)));
  EGFEM_CUDA_TRY(cudaMalloc(k, sizeof(uint32_t) * std::max<int64_t>(m, 1)));
  EGFEM_CUDA_TRY(cudaMalloc(val, sizeof(double) * std::max<int64_t>(m, 1)));
  P.key = *key;
  P.kout = *k;
  P.val = *val;
  if (t->n_cells > 0) {
    k_element_triples<<<nblk(t->n_cells, 128), 128>>>(P);
    count_launch();
    EGFEM_CUDA_TRY(cudaGetLastError());
  }
  *m_out = m;
  return EGFEM_OK;
}

// Sort, merge and compress the emitted triples into the CSF handle.  Takes
// ownership of (and frees) the three input arrays.
egfem_status build_from_triples(egfem_tensor* t, int64_t m, uint64_t* d_key_ij, uint32_t* d_k, double* d_val) {
  DBuf<uint64_t> key_ij;
  key_ij.p = d_key_ij;
  DBuf<uint32_t> kin;
  kin.p = d_k;
  DBuf<double> vin;
  vin.p = d_val;
  if (m >= (int64_t(1) << 32)) {
    set_error("more than 2^32 emitted triples");
    return EGFEM_ERR_INDEX_OVERFLOW;
  }
  const int ij_bits = bits_for((uint64_t)t->n_u * (uint64_t)t->n_u - 1);
  const int k_bits = bits_for((uint64_t)std::max<int64_t>(t->n_f - 1, 1));
  DBuf<uint32_t> idx_a, idx_b;
  EGFEM_CUDA_TRY(idx_a.alloc(m));
  EGFEM_CUDA_TRY(idx_b.alloc(m));
  if (m > 0) {
    k_iota<<<nblk(m), 256>>>(idx_a.p, m);
    count_launch();
  }
  size_t tmp_bytes = 0;
  DBuf<char> tmp;
  if (m > 0 && ij_bits + k_bits <= 64) {
    DBuf<uint64_t> ka, kb;
    EGFEM_CUDA_TRY(ka.alloc(m));
    EGFEM_CUDA_TRY(kb.alloc(m));
    k_pack_key<<<nblk(m), 256>>>(key_ij.p, kin.p, k_bits, ka.p, m);
    count_launch();
    EGFEM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, ka.p, kb.p, idx_a.p, idx_b.p, m, 0,
                                                   ij_bits + k_bits));
    EGFEM_CUDA_TRY(tmp.alloc((int64_t)tmp_bytes));
    EGFEM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, ka.p, kb.p, idx_a.p, idx_b.p, m, 0,
                                                   ij_bits + k_bits));
    count_launch(4);
    std::swap(idx_a.p, idx_b.p);  // sorted order in idx_a
  } else if (m > 0) {
    // LSD: stable sort by k, then stable sort by (i,j) key.
    DBuf<uint32_t> ks;
    EGFEM_CUDA_TRY(ks.alloc(m));
    EGFEM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin.p, ks.p, idx_a.p, idx_b.p, m, 0, k_bits));
    EGFEM_CUDA_TRY(tmp.alloc((int64_t)tmp_bytes));
    EGFEM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, kin.p, ks.p, idx_a.p, idx_b.p, m, 0, k_bits));
    count_launch(4);
    cudaFree(ks.release());
    DBuf<uint64_t> ka, kb;
    EGFEM_CUDA_TRY(ka.alloc(m));
    EGFEM_CUDA_TRY(kb.alloc(m));
    k_gather<uint64_t><<<nblk(m), 256>>>(key_ij.p, idx_b.p, ka.p, m);
    count_launch();
    size_t tb2 = 0;
    EGFEM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb2, ka.p, kb.p, idx_b.p, idx_a.p, m, 0, ij_bits));
    if (tb2 > tmp_bytes) {
      cudaFree(tmp.release());
      EGFEM_CUDA_TRY(tmp.alloc((int64_t)tb2));
      tmp_bytes = tb2;
    }
    EGFEM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, ka.p, kb.p, idx_b.p, idx_a.p, m, 0, ij_bits));
    count_launch(4);
  }
  cudaFree(tmp.release());
  cudaFree(idx_b.release());
  // gather in sorted order
  DBuf<uint64_t> skey;
  DBuf<uint32_t> sk;
  DBuf<double> sval;
  EGFEM_CUDA_TRY(skey.alloc(m));
  EGFEM_CUDA_TRY(sk.alloc(m));
  EGFEM_CUDA_TRY(sval.alloc(m));
  if (m > 0) {
    k_gather<uint64_t><<<nblk(m), 256>>>(key_ij.p, idx_a.p, skey.p, m);
    k_gather<uint32_t><<<nblk(m), 256>>>(kin.p, idx_a.p, sk.p, m);
    k_gather<double><<<nblk(m), 256>>>(vin.p, idx_a.p, sval.p, m);
    count_launch(3);
  }
  cudaFree(key_ij.release());
  cudaFree(kin.release());
  cudaFree(vin.release());
  cudaFree(idx_a.release());
  EGFEM_CUDA_TRY(cudaGetLastError());

  // unique (i,j,k) runs
  DBuf<int32_t> flag;
  DBuf<int64_t> pos;
  EGFEM_CUDA_TRY(flag.alloc(m));
  EGFEM_CUDA_TRY(pos.alloc(m + 1));
  int64_t nnz = 0;
  if (m > 0) {
    k_unique_flags<<<nblk(m), 256>>>(skey.p, sk.p, flag.p, m);
    count_launch();
    size_t tb = 0;
    EGFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.p, pos.p, m + 0));
    EGFEM_CUDA_TRY(tmp.alloc((int64_t)tb));
    EGFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag.p, pos.p, m));
    count_launch(2);
    cudaFree(tmp.release());
    int64_t last_pos = 0;
    int32_t last_flag = 0;
    EGFEM_CUDA_TRY(cudaMemcpy(&last_pos, pos.p + m - 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
    EGFEM_CUDA_TRY(cudaMemcpy(&last_flag, flag.p + m - 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
    nnz = last_pos + last_flag;
  }
  if (nnz >= (int64_t(1) << 32) - 1) {
    set_error("nnz >= 2^32");
    return EGFEM_ERR_INDEX_OVERFLOW;
  }
  DBuf<int64_t> ustart;
  DBuf<uint64_t> nkey;
  DBuf<double> nval;
  EGFEM_CUDA_TRY(ustart.alloc(nnz + 1));
  EGFEM_CUDA_TRY(nkey.alloc(nnz));
  EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->nz_k, sizeof(uint32_t) * nnz));
  EGFEM_CUDA_TRY(nval.alloc(nnz));
  if (m > 0) {
    k_mark_starts<<<nblk(m), 256>>>(flag.p, pos.p, ustart.p, m);
    k_reduce_runs<<<nblk(nnz), 256>>>(ustart.p, nnz, m, skey.p, sk.p, sval.p, nkey.p, t->nz_k, nval.p);
    count_launch(2);
  }
  cudaFree(skey.release());
  cudaFree(sk.release());
  cudaFree(sval.release());
  cudaFree(ustart.release());
  EGFEM_CUDA_TRY(cudaGetLastError());
  t->nnz = nnz;

  // fibers and rows
  int64_t n_fib = 0;
  DBuf<int64_t> row_cnt;
  EGFEM_CUDA_TRY(row_cnt.alloc(t->n_u + 1));
  EGFEM_CUDA_TRY(cudaMemset(row_cnt.p, 0, sizeof(int64_t) * (t->n_u + 1)));
  if (nnz > 0) {
    k_fiber_flags<<<nblk(nnz), 256>>>(nkey.p, flag.p, nnz);
    count_launch();
    size_t tb = 0;
    EGFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.p, pos.p, nnz));
    EGFEM_CUDA_TRY(tmp.alloc((int64_t)tb));
    EGFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag.p, pos.p, nnz));
    count_launch(2);
    cudaFree(tmp.release());
    int64_t last_pos = 0;
    int32_t last_flag = 0;
    EGFEM_CUDA_TRY(cudaMemcpy(&last_pos, pos.p + nnz - 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
    EGFEM_CUDA_TRY(cudaMemcpy(&last_flag, flag.p + nnz - 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
    n_fib = last_pos + last_flag;
  }
  t->n_fib = n_fib;
  EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->fib_nz, sizeof(uint32_t) * (n_fib + 1)));
  EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->fib_j, sizeof(int32_t) * n_fib));
  EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->row_fib, sizeof(int64_t) * (t->n_u + 1)));
  {
    uint32_t nnz32 = (uint32_t)nnz;
    EGFEM_CUDA_TRY(cudaMemcpy(t->fib_nz + n_fib, &nnz32, sizeof(uint32_t), cudaMemcpyHostToDevice));
  }
  if (nnz > 0) {
    k_fiber_fill<<<nblk(nnz), 256>>>(flag.p, pos.p, nkey.p, t->n_u, nnz, t->fib_nz, t->fib_j, row_cnt.p);
    count_launch();
  }
  {
    size_t tb = 0;
    EGFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, row_cnt.p, t->row_fib, t->n_u + 1));
    EGFEM_CUDA_TRY(tmp.alloc((int64_t)tb));
    EGFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tb, row_cnt.p, t->row_fib, t->n_u + 1));
    count_launch(2);
    cudaFree(tmp.release());
  }
  cudaFree(flag.release());
  cudaFree(pos.release());
  cudaFree(row_cnt.release());

  // P0 W: pack the local index of j in cell k into nz_k
  if (t->has_mesh && t->w_p0) {
    if (t->n_f >= (int64_t(1) << kKShift)) {
      set_error("P0 W with N_f >= 2^28");
      return EGFEM_ERR_INDEX_OVERFLOW;
    }
    DBuf<int> err;
    EGFEM_CUDA_TRY(err.alloc(1));
    EGFEM_CUDA_TRY(cudaMemset(err.p, 0, sizeof(int)));
    if (nnz > 0) {
      k_pack_loc<<<nblk(nnz), 256>>>(nkey.p, t->nz_k, nnz, t->n_u, t->wcell, t->vdofs, t->nV, err.p);
      count_launch();
    }
    int herr = 0;
    EGFEM_CUDA_TRY(cudaMemcpy(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (herr) {
      set_error("P0 W: column not found in cell (inconsistent V/W tables)");
      return EGFEM_ERR_INVALID_ARGUMENT;
    }
  }
  // P0 W: position of k among the cells of row i (the k's of the diagonal fiber (i,i))
  if (t->has_mesh && t->w_p0) {
    EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->nz_aux, nnz));
    DBuf<int> err;
    EGFEM_CUDA_TRY(err.alloc(1));
    EGFEM_CUDA_TRY(cudaMemset(err.p, 0, sizeof(int)));
    if (nnz > 0) {
      k_cell_slot<<<nblk(nnz), 256>>>(nkey.p, nnz, t->n_u, t->row_fib, t->fib_j, t->fib_nz, t->nz_k, t->nV,
                                      t->nz_aux, err.p);
      count_launch();
    }
    int herr = 0;
    EGFEM_CUDA_TRY(cudaMemcpy(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (herr) {
      set_error("P0 W: a vertex lies in more than 255 cells or a row is not (d+1) x cells");
      return EGFEM_ERR_UNSUPPORTED;
    }
  }
  cudaFree(nkey.release());

  // fiber-head flags and the row -> first-nonzero pointer
  if (n_fib > 0) {
    k_heads<<<nblk(n_fib), 256>>>(t->fib_nz, n_fib, t->nz_k);
    count_launch();
  }
  EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->row_nz, sizeof(int64_t) * (t->n_u + 1)));
  k_row_nz<<<nblk(t->n_u + 1), 256>>>(t->row_fib, t->fib_nz, t->n_u, t->row_nz);
  count_launch();

  // values in the handle dtype
  if (t->dtype == EGFEM_F64) {
    EGFEM_CUDA_TRY(dmalloc_padded(&t->nz_val, sizeof(double) * nnz));
    if (nnz > 0) EGFEM_CUDA_TRY(cudaMemcpy(t->nz_val, nval.p, sizeof(double) * nnz, cudaMemcpyDeviceToDevice));
  } else {
    EGFEM_CUDA_TRY(dmalloc_padded(&t->nz_val, sizeof(float) * nnz));
    if (nnz > 0) {
      k_to_f32<<<nblk(nnz), 256>>>(nval.p, (float*)t->nz_val, nnz);
      count_launch();
    }
  }
  EGFEM_CUDA_TRY(cudaGetLastError());

  // tiles: greedy over rows with caps on nonzeros, fibers and rows
  std::vector<int64_t> hrf(t->n_u + 1);
  std::vector<uint32_t> hfn(n_fib + 1);
  EGFEM_CUDA_TRY(cudaMemcpy(hrf.data(), t->row_fib, sizeof(int64_t) * (t->n_u + 1), cudaMemcpyDeviceToHost));
  EGFEM_CUDA_TRY(cudaMemcpy(hfn.data(), t->fib_nz, sizeof(uint32_t) * (n_fib + 1), cudaMemcpyDeviceToHost));
  egfem_status st = make_tiles(t, hrf, hfn);
  if (st) return st;
  if ((st = make_wv_aux(t))) return st;
  if ((st = make_p0_cells(t))) return st;
  if ((st = make_step_plan(t))) return st;
  if ((st = make_dense_blocks(t, hrf))) return st;
  if ((st = make_groups(t, hrf))) return st;
  EGFEM_CUDA_TRY(cudaDeviceSynchronize());
  return EGFEM_OK;
}

// Greedy row tiling (≤ kTileNnz nonzeros, ≤ kTileFib fibers, ≤ kTileRows rows per tile) and
// the per-tile (row, fiber, nonzero) start offsets the persistent kernels read.
egfem_status make_tiles(egfem_tensor* t, const std::vector<int64_t>& hrf, const std::vector<uint32_t>& hfn) {
  std::vector<int64_t> tiles{0};
  int64_t tn = 0, tf = 0, tr = 0;
  int max_rn = 0, max_rf = 0;
  for (int64_t i = 0; i < t->n_u; ++i) {
    const int64_t rf = hrf[i + 1] - hrf[i];
    const int64_t rn = (int64_t)hfn[hrf[i + 1]] - (int64_t)hfn[hrf[i]];
    max_rn = std::max<int>(max_rn, (int)rn);
    max_rf = std::max<int>(max_rf, (int)rf);
    if (rn > kTileNnz || rf > kTileFib) {
      set_error("a row exceeds the kernel tile (" + std::to_string(rn) + " nonzeros, " + std::to_string(rf) +
                " fibers)");
      return EGFEM_ERR_UNSUPPORTED;
    }
    if (tr > 0 && (tn + rn > kTileNnz || tf + rf > kTileFib || tr + 1 > kTileRows)) {
      tiles.push_back(i);
      tn = tf = tr = 0;
    }
    tn += rn;
    tf += rf;
    tr += 1;
  }
  if (t->n_u > 0) tiles.push_back(t->n_u);
  t->max_row_nnz = max_rn;
  t->max_row_fib = max_rf;
  t->n_tiles = (int32_t)(tiles.size() - 1);
  std::vector<int64_t> tf_(tiles.size()), te_(tiles.size());
  for (size_t q = 0; q < tiles.size(); ++q) {
    tf_[q] = hrf[tiles[q]];
    te_[q] = hfn[tf_[q]];
  }
  const size_t nb = sizeof(int64_t) * tiles.size();
  EGFEM_CUDA_TRY(cudaMalloc(&t->tile_row, nb));
  EGFEM_CUDA_TRY(cudaMalloc(&t->tile_fib, nb));
  EGFEM_CUDA_TRY(cudaMalloc(&t->tile_nz, nb));
  EGFEM_CUDA_TRY(cudaMemcpy(t->tile_row, tiles.data(), nb, cudaMemcpyHostToDevice));
  EGFEM_CUDA_TRY(cudaMemcpy(t->tile_fib, tf_.data(), nb, cudaMemcpyHostToDevice));
  EGFEM_CUDA_TRY(cudaMemcpy(t->tile_nz, te_.data(), nb, cudaMemcpyHostToDevice));
  return EGFEM_OK;
}

cudaError_t dmalloc_padded(void** p, size_t bytes) {
  // +64 B: the persistent kernels' 16-byte-aligned bulk copies may over-read a tile's tail.
  return cudaMalloc(p, bytes + 64);
}

// ------------------------------------------------------------------ export
namespace {
__global__ void k_export_nz(const int64_t* row_fib, const int32_t* fib_j, const uint32_t* fib_nz,
                            const uint32_t* nz_k, int64_t n_u, bool p0, const int32_t* wcell, const int32_t* vdofs,
                            int nV, int32_t* t_j, int32_t* t_k, int32_t* slot_ij, int32_t* slot_ik, uint8_t* loc,
                            int64_t* t_row_ptr) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_u) return;
  const int64_t f0 = row_fib[i], f1 = row_fib[i + 1];
  t_row_ptr[i] = fib_nz[f0];
  if (i == n_u - 1) t_row_ptr[n_u] = fib_nz[f1];
  for (int64_t f = f0; f < f1; ++f) {
    for (uint32_t e = fib_nz[f]; e < fib_nz[f + 1]; ++e) {
      uint32_t kk = nz_k[e];
      uint32_t k = kk & (p0 ? kKMask : kKMaskAny);
      if (t_j) t_j[e] = fib_j[f];
      if (t_k) t_k[e] = (int32_t)k;
      if (slot_ij) slot_ij[e] = (int32_t)f;
      if (slot_ik) {
        int64_t lo = f0, hi = f1;  // binary search k among the row's columns
        while (lo < hi) {
          int64_t mid = (lo + hi) / 2;
          if (fib_j[mid] < (int32_t)k) lo = mid + 1; else hi = mid;
        }
        slot_ik[e] = (lo < f1 && fib_j[lo] == (int32_t)k) ? (int32_t)lo : -1;
      }
      if (loc) {
        int64_t c = wcell[k];
        int li = 0;
        for (int a = 0; a < nV; ++a)
          if (vdofs[c * nV + a] == (int32_t)i) li = a;
        loc[e] = (uint8_t)(li | (((kk >> kKShift) & 3u) << 2));
      }
    }
  }
}
}  // namespace

egfem_status export_arrays(const egfem_tensor* t, int64_t* t_row_ptr, int32_t* t_j, int32_t* t_k, void* t_val,
                           int64_t* csr_row_ptr, int32_t* csr_col, int32_t* slot_ij, int32_t* slot_ik,
                           uint8_t* loc) {
  const int64_t nnz = t->nnz;
  DBuf<int32_t> dj, dk, dsij, dsik;
  DBuf<uint8_t> dloc;
  DBuf<int64_t> drp;
  EGFEM_CUDA_TRY(drp.alloc(t->n_u + 1));
  if (t_j) EGFEM_CUDA_TRY(dj.alloc(nnz));
  if (t_k) EGFEM_CUDA_TRY(dk.alloc(nnz));
  if (slot_ij) EGFEM_CUDA_TRY(dsij.alloc(nnz));
  if (slot_ik) EGFEM_CUDA_TRY(dsik.alloc(nnz));
  if (loc) EGFEM_CUDA_TRY(dloc.alloc(nnz));
  if (t->n_u > 0) {
    k_export_nz<<<nblk(t->n_u), 256>>>(t->row_fib, t->fib_j, t->fib_nz, t->nz_k, t->n_u, t->w_p0 && t->has_mesh,
                                       t->wcell, t->vdofs, t->nV, dj.p, dk.p, dsij.p, dsik.p, dloc.p, drp.p);
    count_launch();
  } else {
    EGFEM_CUDA_TRY(cudaMemset(drp.p, 0, sizeof(int64_t)));
  }
  EGFEM_CUDA_TRY(cudaGetLastError());
  EGFEM_CUDA_TRY(cudaDeviceSynchronize());
  if (t_row_ptr) EGFEM_CUDA_TRY(cudaMemcpy(t_row_ptr, drp.p, sizeof(int64_t) * (t->n_u + 1), cudaMemcpyDeviceToHost));
  if (t_j) EGFEM_CUDA_TRY(cudaMemcpy(t_j, dj.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
  if (t_k) EGFEM_CUDA_TRY(cudaMemcpy(t_k, dk.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
  if (t_val)
    EGFEM_CUDA_TRY(cudaMemcpy(t_val, t->nz_val, (t->dtype == EGFEM_F64 ? 8 : 4) * nnz, cudaMemcpyDeviceToHost));
  if (csr_row_ptr)
    EGFEM_CUDA_TRY(cudaMemcpy(csr_row_ptr, t->row_fib, sizeof(int64_t) * (t->n_u + 1), cudaMemcpyDeviceToHost));
  if (csr_col) EGFEM_CUDA_TRY(cudaMemcpy(csr_col, t->fib_j, sizeof(int32_t) * t->n_fib, cudaMemcpyDeviceToHost));
  if (slot_ij) EGFEM_CUDA_TRY(cudaMemcpy(slot_ij, dsij.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
  if (slot_ik) EGFEM_CUDA_TRY(cudaMemcpy(slot_ik, dsik.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
  if (loc) EGFEM_CUDA_TRY(cudaMemcpy(loc, dloc.p, nnz, cudaMemcpyDeviceToHost));
  return EGFEM_OK;
}

void free_tensor(egfem_tensor* t) {
  void* ptrs[] = {t->row_fib, t->row_nz, t->fib_j, t->fib_nz, t->nz_k, t->nz_val, t->nz_aux, t->nz_kpos, t->fib_kr, t->ck_k, t->ck_val, t->ck_b, t->ck_m, t->ck_kb, t->blk_off, t->blk, t->blk_sym, t->dense_rows,
                  t->tile_row, t->tile_fib, t->tile_nz, t->coords, t->coords4, t->coordsf, t->cells, t->vdofs, t->wdofs, t->wcell, t->wpts, t->gcls, t->gtab};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  free_group_plan(t->grp);
  t->grp = nullptr;
  free_step_plan(t->step);
  t->step = nullptr;
}

}  // namespace egfem

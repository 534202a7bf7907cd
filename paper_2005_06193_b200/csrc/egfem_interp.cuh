// Step (1) of the gradient kinds, shared by the interp kernel (egfem_kernels.cu) and the
// single-pass Newton step kernel (egfem_cells.cu).  Internal to libegfem.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#ifndef EGFEM_INTERP_PFD
#define EGFEM_INTERP_PFD 0  // A/B: L2 prefetch of the cell records this many grid strides ahead (0 = off)
#endif
#ifndef EGFEM_INTERP_EF
#define EGFEM_INTERP_EF 0  // A/B: 1 = cell records loaded and Newton records stored L2 evict-first, 2 = stores only
#endif
#ifndef EGFEM_INTERP_LEAN
#define EGFEM_INTERP_LEAN 1  // lean 3D gradient form (A/B switch; 0: ∇λ_a formed first)
#endif

namespace egfem {
namespace ip {

// GRADPOW_P0: g_K = Σ_a u_{v_a} ∇λ_a (Π_∇u ·₂ u at the cell's DOF), w_K = ‖g_K‖^{p−2},
// ∂w_K/∂u_{v_m} = (p−2)‖g‖^{p−4} g·∇λ_m (reading C11); chain[K] = [w_K, ∂w_K/∂u_{v_0}
// .. ∂w_K/∂u_{v_{d−1}}] (packed: the last derivative is −Σ of the others).
// Thread per cell; 3D reads the cell as one int4 and each vertex as two double2 from the
// 32-byte padded coordinate array, and writes the chain row as two 16-byte stores.
template <int D>
struct CellIdx {
  int32_t v[D + 1];
};
template <int D>
__device__ __forceinline__ CellIdx<D> load_cidx(const int32_t* __restrict__ t, int64_t c) {
  CellIdx<D> r;
  if constexpr (D == 3 && EGFEM_INTERP_EF == 1) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int4 q;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
        : "l"(reinterpret_cast<const int4*>(t) + c), "l"(pol));
    r.v[0] = q.x;
    r.v[1] = q.y;
    r.v[2] = q.z;
    r.v[3] = q.w;
  } else if constexpr (D == 3) {
    const int4 q = __ldg(reinterpret_cast<const int4*>(t) + c);
    r.v[0] = q.x;
    r.v[1] = q.y;
    r.v[2] = q.z;
    r.v[3] = q.w;
  } else {
#pragma unroll
    for (int a = 0; a <= D; ++a) r.v[a] = __ldg(t + c * (D + 1) + a);
  }
  return r;
}

// One cell's gathered inputs: vertex coordinates and u at its V DOFs.
template <typename S, int D>
struct CellIn {
  double x[D + 1][D];
  double uv[D + 1];
};
template <typename S, int D, bool SAME, bool CF>
__device__ __forceinline__ void gather_cell(const double* __restrict__ coords, const float* __restrict__ coordsf,
                                            const CellIdx<D>& cv, const CellIdx<D>& dv, const S* __restrict__ u,
                                            CellIn<S, D>& in) {
#pragma unroll
  for (int a = 0; a <= D; ++a) {
    const int64_t v = cv.v[a];
    if constexpr (D == 3 && CF) {  // exact float copy of the coordinates: one 16-byte load
      const float4 q = __ldg(reinterpret_cast<const float4*>(coordsf) + v);
      in.x[a][0] = (double)q.x;
      in.x[a][1] = (double)q.y;
      in.x[a][2] = (double)q.z;
    } else if constexpr (D == 2 && CF) {  // exact float copy: one 8-byte load
      const float2 q = __ldg(reinterpret_cast<const float2*>(coordsf) + v);
      in.x[a][0] = (double)q.x;
      in.x[a][1] = (double)q.y;
    } else if constexpr (D == 3) {
      const double2 xy = __ldg(reinterpret_cast<const double2*>(coords + v * 4));
      in.x[a][0] = xy.x;
      in.x[a][1] = xy.y;
      in.x[a][2] = __ldg(coords + v * 4 + 2);
    } else if constexpr (D == 2) {
      const double2 xy = __ldg(reinterpret_cast<const double2*>(coords + v * 2));
      in.x[a][0] = xy.x;
      in.x[a][1] = xy.y;
    } else {
      in.x[a][0] = __ldg(coords + v);
    }
    in.uv[a] = (double)__ldg(u + dv.v[a]);
  }
}

// 3D cell geometry from the edge vectors e_a = x_{a+1} − x_0: the cofactor vectors c_a (∇λ_{a+1} =
// c_a / det) and 1/det, with every rounding explicit — the geometry-class table (kernel k_geo_table)
// evaluates the same function on a class's edge vectors and must match the per-cell path bit for bit
__device__ __forceinline__ void cof3(const double (&e)[3][3], double (&cc)[3][3], double& inv3) {
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int q1 = (q + 1) % 3, q2 = (q + 2) % 3;
    cc[0][q] = __fma_rn(e[1][q1], e[2][q2], -__dmul_rn(e[1][q2], e[2][q1]));
    cc[1][q] = __fma_rn(e[2][q1], e[0][q2], -__dmul_rn(e[2][q2], e[0][q1]));
    cc[2][q] = __fma_rn(e[0][q1], e[1][q2], -__dmul_rn(e[0][q2], e[1][q1]));
  }
  inv3 = 1.0 / __fma_rn(e[0][2], cc[0][2], __fma_rn(e[0][1], cc[0][1], __dmul_rn(e[0][0], cc[0][0])));
}

// GEO: the cell's geometry (cc, inv3 as 10 values, `geo[a * 3 + q]`, `geo[9]`) comes from its
// geometry class instead of its vertex coordinates (3D lean form only; in.x is not read)
template <typename S, int D, bool IOTA, bool GEO = false>
__device__ __forceinline__ void gradpow_cell(const CellIn<S, D>& in, int64_t c, const int32_t* __restrict__ wdofs,
                                             S* __restrict__ w, S* __restrict__ chain, double p, bool minsurf,
                                             int nw, const double* geo = nullptr) {
  static_assert(!GEO || (D == 3 && EGFEM_INTERP_LEAN), "geometry classes: 3D lean form");
  const auto& x = in.x;
  const auto& uv = in.uv;
  // barycentric gradients of vertices 1..D from the edge vectors e_a = x_a − x_0
  double g[D + 1][D];
  if constexpr (D == 1) {
    g[1][0] = 1.0 / (x[1][0] - x[0][0]);
  } else if constexpr (D == 2) {
    const double e1x = x[1][0] - x[0][0], e1y = x[1][1] - x[0][1];
    const double e2x = x[2][0] - x[0][0], e2y = x[2][1] - x[0][1];
    const double inv = 1.0 / (e1x * e2y - e1y * e2x);
    g[1][0] = e2y * inv;
    g[1][1] = -e2x * inv;
    g[2][0] = -e1y * inv;
    g[2][1] = e1x * inv;
  } else if constexpr (EGFEM_INTERP_LEAN) {
    // (lean 3D form below, after the generic block)
  } else {
    double e[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int q = 0; q < 3; ++q) e[a][q] = x[a + 1][q] - x[0][q];
    const double c23[3] = {e[1][1] * e[2][2] - e[1][2] * e[2][1], e[1][2] * e[2][0] - e[1][0] * e[2][2],
                           e[1][0] * e[2][1] - e[1][1] * e[2][0]};
    const double c31[3] = {e[2][1] * e[0][2] - e[2][2] * e[0][1], e[2][2] * e[0][0] - e[2][0] * e[0][2],
                           e[2][0] * e[0][1] - e[2][1] * e[0][0]};
    const double c12[3] = {e[0][1] * e[1][2] - e[0][2] * e[1][1], e[0][2] * e[1][0] - e[0][0] * e[1][2],
                           e[0][0] * e[1][1] - e[0][1] * e[1][0]};
    const double inv = 1.0 / (e[0][0] * c23[0] + e[0][1] * c23[1] + e[0][2] * c23[2]);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      g[1][q] = c23[q] * inv;
      g[2][q] = c31[q] * inv;
      g[3][q] = c12[q] * inv;
    }
  }
  double gu[D];
  // lean 3D: ∇λ_a = c_a / det (a = 1..3), Σ_a ∇λ_a = 0, so ∇u_h = (1/det) Σ_{a≥1} (u_a − u_0) c_a and
  // the derivative record needs only gu·c_a
  double cc[EGFEM_INTERP_LEAN && D == 3 ? 3 : 1][3], inv3 = 0.0;
  if constexpr (EGFEM_INTERP_LEAN && D == 3) {
    if constexpr (GEO) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int q = 0; q < 3; ++q) cc[a][q] = geo[a * 3 + q];
      inv3 = geo[9];
    } else {
      double e[3][3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int q = 0; q < 3; ++q) e[a][q] = x[a + 1][q] - x[0][q];
      cof3(e, cc, inv3);
    }
    const double d1 = uv[1] - uv[0], d2 = uv[2] - uv[0], d3 = uv[3] - uv[0];
#pragma unroll
    for (int q = 0; q < 3; ++q)
      gu[q] = __dmul_rn(inv3, __fma_rn(d3, cc[2][q], __fma_rn(d2, cc[1][q], __dmul_rn(d1, cc[0][q]))));
  } else {
#pragma unroll
    for (int q = 0; q < D; ++q) {
      double s = 0.0;
#pragma unroll
      for (int a = 1; a <= D; ++a) s += g[a][q];
      g[0][q] = -s;
    }
#pragma unroll
    for (int q = 0; q < D; ++q) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a <= D; ++a) s += uv[a] * g[a][q];
      gu[q] = s;
    }
  }
  double gg = 0.0;
#pragma unroll
  for (int q = 0; q < D; ++q) gg = __fma_rn(gu[q], gu[q], gg);
  double wk, fac;
  if (minsurf) {  // a = (1 + ‖g‖²)^{−1/2}, ∂a/∂u_m = −(1 + ‖g‖²)^{−3/2} g·∇λ_m
    wk = 1.0 / sqrt(1.0 + gg);
    fac = -(wk * wk * wk);
  } else if (p == 4.0) {
    wk = gg;
    fac = 2.0;
  } else if (p == 3.0) {
    const double nrm = sqrt(gg);
    wk = nrm;
    fac = gg > 0.0 ? 1.0 / nrm : 0.0;
  } else if (p == 2.0) {
    wk = 1.0;
    fac = 0.0;
  } else {
    wk = pow(gg, 0.5 * (p - 2.0));
    fac = gg > 0.0 ? (p - 2.0) * pow(gg, 0.5 * (p - 4.0)) : 0.0;
  }
  // the packed chain record (include/egfem.h egfem_interp): [w_K, ∂w/∂u_{v_0} .. ∂w/∂u_{v_{d−1}}];
  // ∂w/∂u_{v_d} = −Σ_{m<d} (Σ_m ∇λ_m = 0), rebuilt by the Jacobian kernels — so the Newton kernel
  // reads w and D_u w of a cell with one gather
  S dm[D + 1];
  if (chain) {
    dm[0] = (S)wk;
    if constexpr (EGFEM_INTERP_LEAN && D == 3) {  // D_a = fac gu·∇λ_a, a = 1..3; D_0 = −(D_1 + D_2 + D_3)
      const double f = fac * inv3;
      double dv[3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
        dv[a] = __dmul_rn(f, __fma_rn(gu[2], cc[a][2], __fma_rn(gu[1], cc[a][1], __dmul_rn(gu[0], cc[a][0]))));
      dm[1] = (S)(-(dv[0] + dv[1] + dv[2]));
      dm[2] = (S)dv[0];
      dm[3] = (S)dv[1];
    } else {
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < D; ++q) s += gu[q] * g[a][q];
        dm[a + 1] = (S)(fac * s);
      }
    }
  }
  // the cell's W DOFs (P0: one; QUAD: N_q points, ∇u_h is constant on the cell)
  if (IOTA) nw = 1;  // canonical P0 (the IOTA instance is only launched for it)
  for (int l = 0; l < nw; ++l) {
    const int64_t K = IOTA ? c : (int64_t)__ldg(wdofs + c * nw + l);
    if (w) w[K] = (S)wk;  // NULL: w_K is kept in the packed record only (include/egfem.h egfem_interp)
    if (chain) {
      if constexpr (D == 3 && sizeof(S) == 8) {  // one 32-byte store (sm_100 256-bit STG) when aligned
        if ((reinterpret_cast<uintptr_t>(chain) & 31u) == 0) {
          if constexpr (EGFEM_INTERP_EF != 0)
            asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(chain + K * 4), "d"(dm[0]),
                         "d"(dm[1]), "d"(dm[2]), "d"(dm[3])
                         : "memory");
          else
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(chain + K * 4), "d"(dm[0]), "d"(dm[1]),
                         "d"(dm[2]), "d"(dm[3])
                         : "memory");
        } else {  // the API's 16-byte alignment
          reinterpret_cast<double2*>(chain + K * 4)[0] = make_double2(dm[0], dm[1]);
          reinterpret_cast<double2*>(chain + K * 4)[1] = make_double2(dm[2], dm[3]);
        }
      } else if constexpr (D == 3) {
        reinterpret_cast<float4*>(chain)[K] = make_float4(dm[0], dm[1], dm[2], dm[3]);
      } else {
#pragma unroll
        for (int a = 0; a <= D; ++a) chain[K * (D + 1) + a] = dm[a];
      }
    }
  }
}

// Cells c, c + stride, ... < cend of one thread, software-pipelined: the cell record is loaded
// two cells ahead and the next cell's vertex coordinates and u one cell ahead, so the dependent
// record → coordinates gather chain overlaps the current cell's arithmetic instead of stalling.
template <typename S, int D, bool SAME, bool IOTA, bool CF>
__device__ __forceinline__ void interp_cells(const double* __restrict__ coords, const float* __restrict__ coordsf,
                                             const int32_t* __restrict__ cells, const int32_t* __restrict__ vdofs,
                                             const int32_t* __restrict__ wdofs, int64_t c, int64_t cend,
                                             int64_t stride, const S* __restrict__ u, S* __restrict__ w,
                                             S* __restrict__ chain, double p, bool minsurf, int nw) {
  if (c >= cend) return;
  auto idx = [&](int64_t cc, CellIdx<D>& cv, CellIdx<D>& dv) {
    const int64_t q = cc < cend ? cc : c;  // clamped: a valid record, never used
    cv = load_cidx<D>(cells, q);
    dv = SAME ? cv : load_cidx<D>(vdofs, q);
  };
  CellIdx<D> cv1, dv1, cv2, dv2;
  idx(c, cv1, dv1);
  CellIn<S, D> cur;
  gather_cell<S, D, SAME, CF>(coords, coordsf, cv1, dv1, u, cur);
  idx(c + stride, cv2, dv2);
  for (; c < cend; c += stride) {
    CellIn<S, D> nxt;
    gather_cell<S, D, SAME, CF>(coords, coordsf, cv2, dv2, u, nxt);  // next cell's gathers in flight
    idx(c + 2 * stride, cv2, dv2);                                    // record two cells ahead
    gradpow_cell<S, D, IOTA>(cur, c, wdofs, w, chain, p, minsurf, nw);
    cur = nxt;
  }
}

// Geometry classes (3D, canonical P1 V / P0 W): cells whose edge vectors are bitwise equal share
// one (cc, inv3) entry of the class table `sg` (shared memory, entry k at sg[v * nk + k], v < 10),
// so a cell needs its class byte and u at its vertices only — no coordinate gathers and no
// cofactor arithmetic (SG: the table staged in shared memory, else read through L1 from global).
// Same pipeline as interp_cells: the cell record two cells ahead, the u
// gathers and the class byte one cell ahead.
template <typename S, bool SG>
__device__ __forceinline__ void interp_cells_geo(const uint8_t* __restrict__ gcls, const double* sg, int nk,
                                                 const int32_t* __restrict__ cells, int64_t c, int64_t cend,
                                                 int64_t stride, const S* __restrict__ u, S* __restrict__ w,
                                                 S* __restrict__ chain, double p, bool minsurf) {
  if (c >= cend) return;
  auto idx = [&](int64_t cc) { return load_cidx<3>(cells, cc < cend ? cc : c); };
  auto gather = [&](const CellIdx<3>& cv, int64_t cc, CellIn<S, 3>& in, int& k) {
#pragma unroll
    for (int a = 0; a <= 3; ++a) in.uv[a] = (double)__ldg(u + cv.v[a]);
    k = __ldg(gcls + (cc < cend ? cc : c));
  };
  CellIdx<3> cv2 = idx(c);
  CellIn<S, 3> cur;
  int kc;
  gather(cv2, c, cur, kc);
  cv2 = idx(c + stride);
  for (; c < cend; c += stride) {
    CellIn<S, 3> nxt;
    int kn;
    gather(cv2, c + stride, nxt, kn);
    cv2 = idx(c + 2 * stride);
    if constexpr (EGFEM_INTERP_PFD > 0) {
      const int64_t cp = c + (int64_t)EGFEM_INTERP_PFD * stride;
      if (cp < cend) asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const int4*>(cells) + cp));
    }
    double geo[10];
#pragma unroll
    for (int v = 0; v < 10; ++v) geo[v] = SG ? sg[v * nk + kc] : __ldg(sg + v * nk + kc);
    gradpow_cell<S, 3, true, true>(cur, c, nullptr, w, chain, p, minsurf, 1, geo);
    cur = nxt;
    kc = kn;
  }
}

}  // namespace ip
}  // namespace egfem

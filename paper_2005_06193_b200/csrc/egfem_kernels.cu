// Per-iteration kernels of libegfem.so (B200 / sm_100a).
//
//   k_interp_*  step (1): w = f(Π_u u, Π_∇u ·₂ u) pointwise at the W-DOFs
//                — one thread per W-DOF / cell.
//   k_tile      steps (2)+(3): r = T:(u⊗w) and the CSR values of
//               A = T·w or J = T·w + (T·₂u)·D_u w.
//               One CTA owns one tile of whole rows: the tile's (k, value) stream is
//               read once with streaming (evict-first) loads, w is gathered through
//               L1/L2, and every reduction (fiber, row, Newton chain) runs in
//               shared memory in a fixed order — no floating-point atomics.
//   k_batched   step (2) for B independent (u, w) pairs: the tile's nonzeros are
//               staged in shared memory once and reused by every pair.
// HBM-bound sparse contractions: no tensor cores.
#include <algorithm>
#include <cstdlib>

#include "egfem_internal.cuh"
#include "egfem_interp.cuh"

namespace egfem {
namespace {

inline int nblk(int64_t n, int t = 256) { return (int)((n + t - 1) / t); }

// Streaming 32/64-bit loads for data touched exactly once (T's k and values).
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) { return __ldcs(p); }
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }

template <typename S>
__device__ __forceinline__ S ld_ro(const S* p) {
  return __ldg(p);
}

// ------------------------------------------------------------------ interp
template <typename S>
__global__ void k_interp_copy(const S* __restrict__ u, S* __restrict__ w, int64_t n, int mode, double pk) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    S x = u[i];
    w[i] = mode == 0 ? x : (mode == 1 ? x * x : S(1) / (S(pk) + x));  // IDENTITY, SQUARE, RECIPROCAL
  }
}

// Grid-stride over the cells, one thread per cell (egfem_interp.cuh interp_cells).
template <typename S, int D, bool SAME, bool IOTA, bool CF>
__global__ void __launch_bounds__(128) k_interp_gradpow(const double* __restrict__ coords, const float* __restrict__ coordsf,
                                 const int32_t* __restrict__ cells,
                                 const int32_t* __restrict__ vdofs, const int32_t* __restrict__ wdofs, int64_t n_cells,
                                 const S* __restrict__ u, S* __restrict__ w, S* __restrict__ chain, double p,
                                 bool minsurf, int nw) {
  ip::interp_cells<S, D, SAME, IOTA, CF>(coords, coordsf, cells, vdofs, wdofs,
                                         (int64_t)blockIdx.x * blockDim.x + threadIdx.x, n_cells,
                                         (int64_t)gridDim.x * blockDim.x, u, w, chain, p, minsurf, nw);
}

// Geometry-class variant (3D, canonical P1 V / P0 W; egfem_interp.cuh interp_cells_geo): the class
// table (cc, inv3 of each class, 10 x nk values, entry-major by value) is staged once per CTA.
// fp32: the interp is FP64-bound (its geometry is fp64) and the class table removes the cofactor
// arithmetic — cfg4 0.127 -> 0.097 ms; fp64 (write-heavy: the 32-byte record) 0.137 -> 0.134 ms at
// 6 CTAs per SM.  SG = false reads the table through L1 (measured slower: fp32 0.105 ms).
template <typename S, bool SG>
__device__ __forceinline__ void geo_body(const double* __restrict__ gtab, int nk, const uint8_t* __restrict__ gcls,
                                         const int32_t* __restrict__ cells, int64_t n_cells, const S* __restrict__ u,
                                         S* __restrict__ w, S* __restrict__ chain, double p, bool minsurf) {
  __shared__ double sg[SG ? 10 * kMaxGeoClasses : 1];
  if constexpr (SG) {
    for (int i = threadIdx.x; i < 10 * nk; i += blockDim.x) sg[i] = gtab[i];
    __syncthreads();
  }
  ip::interp_cells_geo<S, SG>(gcls, SG ? sg : gtab, nk, cells, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, n_cells,
                              (int64_t)gridDim.x * blockDim.x, u, w, chain, p, minsurf);
}
// fp64 at 6 CTAs per SM (80 registers, 32 bytes of spill stores): 0.134 ms vs 0.137 gathering and
// 0.142 / 0.164 / 0.189 ms at 96 / unbounded / 64 registers; fp32 without a minimum (80 registers):
// 0.097 ms vs 0.100 at 6 per SM (profiles/r2_geo_minb_ab_v1.jsonl)
template <typename S, bool SG>
__global__ void __launch_bounds__(128) k_interp_gradpow_geo(const double* __restrict__ gtab, int nk,
                                                            const uint8_t* __restrict__ gcls,
                                                            const int32_t* __restrict__ cells, int64_t n_cells,
                                                            const S* __restrict__ u, S* __restrict__ w,
                                                            S* __restrict__ chain, double p, bool minsurf) {
  geo_body<S, SG>(gtab, nk, gcls, cells, n_cells, u, w, chain, p, minsurf);
}
template <typename S, bool SG>
__global__ void __launch_bounds__(128, 6) k_interp_gradpow_geo6(const double* __restrict__ gtab, int nk,
                                                                const uint8_t* __restrict__ gcls,
                                                                const int32_t* __restrict__ cells, int64_t n_cells,
                                                                const S* __restrict__ u, S* __restrict__ w,
                                                                S* __restrict__ chain, double p, bool minsurf) {
  geo_body<S, SG>(gtab, nk, gcls, cells, n_cells, u, w, chain, p, minsurf);
}

// Value kinds at the W DOFs of a cell-wise W (V = P1): u_h(x_l) = Σ_a λ_a(x_l) u_a with λ(x_l)
// from wpts (P0: the centroid; QUAD: the rule's points), then
//   mode 0 RECIPROCAL: w = 1/(k + u_h), ∂w/∂u_m = −w² λ_m
//   mode 1 SQUARE:     w = u_h²,        ∂w/∂u_m = 2 u_h λ_m
template <typename S>
__global__ void k_interp_points(const int32_t* __restrict__ vdofs, const int32_t* __restrict__ wdofs,
                                const double* __restrict__ wpts, int64_t n_cells, int d1, int nw,
                                const S* __restrict__ u, S* __restrict__ w, S* __restrict__ chain, int mode,
                                double pk) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  double uv[4];
  for (int a = 0; a < d1; ++a) uv[a] = (double)__ldg(u + vdofs[c * d1 + a]);
  for (int l = 0; l < nw; ++l) {
    const double* lam = wpts + l * d1;
    double uh = 0.0;
    for (int a = 0; a < d1; ++a) uh += lam[a] * uv[a];
    double f, df;
    if (mode == 0) {
      f = 1.0 / (pk + uh);
      df = -(f * f);
    } else {
      f = uh * uh;
      df = 2.0 * uh;
    }
    const int64_t K = wdofs[c * nw + l];
    w[K] = (S)f;
    if (chain)
      for (int a = 0; a < d1; ++a) chain[K * d1 + a] = (S)(df * lam[a]);
  }
}

// The same with canonical cell-wise numbering (W DOF l of cell c is c·nw + l): a CTA's cells own
// one contiguous span of w and of the chain, so each thread computes its cell's points into
// shared memory and the CTA writes both spans out coalesced (the per-thread rows of the kernel
// above are nw and nw·(d+1) values apart between neighbouring threads).
template <typename S>
__global__ void __launch_bounds__(128) k_interp_points_blk(const int32_t* __restrict__ vdofs,
                                                           const double* __restrict__ wpts, int64_t n_cells, int d1,
                                                           int nw, const S* __restrict__ u, S* __restrict__ w,
                                                           S* __restrict__ chain, int mode, double pk) {
  extern __shared__ __align__(16) unsigned char smem_pts[];
  S* s_w = reinterpret_cast<S*>(smem_pts);
  S* s_c = s_w + 128 * nw;
  const int64_t c0 = (int64_t)blockIdx.x * 128;
  const int nc = (int)min((int64_t)128, n_cells - c0);
  const int tid = threadIdx.x;
  if (tid < nc) {
    const int64_t c = c0 + tid;
    double uv[4];
    for (int a = 0; a < d1; ++a) uv[a] = (double)__ldg(u + __ldg(vdofs + c * d1 + a));
    for (int l = 0; l < nw; ++l) {
      const double* lam = wpts + l * d1;
      double uh = 0.0;
      for (int a = 0; a < d1; ++a) uh += lam[a] * uv[a];
      double f, df;
      if (mode == 0) {
        f = 1.0 / (pk + uh);
        df = -(f * f);
      } else {
        f = uh * uh;
        df = 2.0 * uh;
      }
      s_w[tid * nw + l] = (S)f;
      if (chain)
        for (int a = 0; a < d1; ++a) s_c[(tid * nw + l) * d1 + a] = (S)(df * lam[a]);
    }
  }
  __syncthreads();
  S* wo = w + c0 * nw;
  for (int x = tid; x < nc * nw; x += 128) wo[x] = s_w[x];
  if (chain) {
    S* co = chain + c0 * nw * d1;
    for (int x = tid; x < nc * nw * d1; x += 128) co[x] = s_c[x];
  }
}

// P1 → P2 interpolant squared: vertex DOFs u_v², edge DOFs ((u_a + u_b)/2)².
template <typename S>
__global__ void k_interp_p1p2sq(const int32_t* __restrict__ vdofs, const int32_t* __restrict__ wdofs, int64_t n_cells,
                                const S* __restrict__ u, S* __restrict__ w) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  double uv[3];
  for (int a = 0; a < 3; ++a) uv[a] = (double)u[vdofs[c * 3 + a]];
  const double val[6] = {uv[0], uv[1], uv[2], 0.5 * (uv[0] + uv[1]), 0.5 * (uv[1] + uv[2]), 0.5 * (uv[2] + uv[0])};
  for (int l = 0; l < 6; ++l) w[wdofs[c * 6 + l]] = (S)(val[l] * val[l]);  // identical values from every cell
}

// ------------------------------------------------------------------ tile kernel
// Persistent CTAs walk the row tiles t = blockIdx.x + q·gridDim.x.  Per tile, one
// thread issues TMA 1D bulk copies (cp.async.bulk, L2 evict-first) of the tile's slices
// of row_fib, fib_nz, fib_j, nz_k, nz_val (and the P0 cell slots) into a stage of an
// NS-deep shared-memory ring, completing on an mbarrier; one tile ahead, every thread
// gathers the tile's w_k (and D_u w, u_j) with cp.async into the same stage.  The CTA
// meanwhile reduces the current tile from shared memory:
//   phase B (thread per fiber)  a_f = Σ_k T_ijk w_k     (Picard value of CSR slot f)
//                               fv_f = a_f u_j;  P0 Newton: B-parts T_ijK u_j
//   phase C (thread per row / fiber)  r_i = Σ_f fv_f;  Newton chain terms.
// All sums run in a fixed order: bitwise reproducible, no floating-point atomics.
enum { kJacNone = 0, kJacPicard = 1, kJacNewtonWV = 2, kJacNewtonP0 = 3 };

template <typename S>
struct TileArgs {
  const int64_t* tile_row;
  const int64_t* tile_fib;
  const int64_t* tile_nz;
  int32_t n_tiles;
  const int64_t* row_fib;
  const int32_t* fib_j;
  const uint32_t* fib_nz;
  const uint32_t* nz_k;
  const S* nz_val;
  const uint8_t* nz_aux;
  const S* u;
  const S* w;
  const S* chain;
  S* r;
  S* csr;
  int d1;       // d+1 (GRADPOW chain stride)
  int packed;   // P0 Newton: packed chain record [w, D_0 .. D_{d−1}], D_d = −Σ (gradient kinds)
  int dmode;    // W = V Newton factor ∂w_m/∂u_m: 0 → 1, 1 → 2u_m (SQUARE), 2 → −1/(pk+u_m)² (RECIPROCAL)
  double pk;
  uint32_t kmask;  // kKMask for P0 W (loc bits), ~0 otherwise
};

__host__ __device__ constexpr int al16(int x) { return (x + 15) & ~15; }
__host__ __device__ constexpr int al128(int x) { return (x + 127) & ~127; }

template <typename S, bool DO_R, int JAC>
struct TileLayout {
  static constexpr bool kP0 = JAC == kJacNewtonP0;
  static constexpr bool kWV = JAC == kJacNewtonWV;
  static constexpr bool kNeedU = DO_R || kWV || kP0;
  static constexpr bool kFrow = kWV || kP0;
  static constexpr int NS = kP0 ? 2 : 3;  // pipeline depth (stages)
  static constexpr int SZ = (int)sizeof(S);
  // stage (bulk-copied slices carry up to 15 B of alignment slack at each end)
  static constexpr int o_rf = 0;
  static constexpr int o_fnz = o_rf + al16((kTileRows + 1) * 8 + 32);
  static constexpr int o_fj = o_fnz + al16((kTileFib + 1) * 4 + 32);
  static constexpr int o_k = o_fj + al16(kTileFib * 4 + 32);
  static constexpr int o_val = o_k + al16(kTileNnz * 4 + 32);
  static constexpr int o_aux = o_val + al16(kTileNnz * SZ + 32);
  static constexpr int o_w = o_aux + (kP0 ? al16(kTileNnz + 32) : 0);
  static constexpr int o_d = o_w + al16(kTileNnz * SZ);
  static constexpr int o_uj = o_d + (kP0 ? al16(kTileNnz * SZ) : 0);
  static constexpr int o_frow = o_uj + (kNeedU ? al16(kTileFib * SZ) : 0);
  static constexpr int stage = al128(o_frow + (kFrow ? al16(kTileFib * 2) : 0));
  // CTA work arrays after the ring
  static constexpr int o_fv = NS * stage;
  static constexpr int o_bp = o_fv + (DO_R ? al16(kTileFib * SZ) : 0);
  static constexpr int o_bar = al16(o_bp + (kP0 ? kTileNnz * SZ : 0));
  static constexpr int bytes = o_bar + NS * 8;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void cp_async_s(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_s(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 16-byte aligned span [align_down(p), align_up(p + bytes)) of a global array.
struct Span {
  const char* src;
  uint32_t bytes;
  int shift;  // elements between the span start and p
};
template <typename T>
__device__ __forceinline__ Span span_of(const T* p, int64_t n) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t lo = a & ~uintptr_t(15);
  const uintptr_t hi = (a + (uintptr_t)n * sizeof(T) + 15) & ~uintptr_t(15);
  return Span{reinterpret_cast<const char*>(lo), (uint32_t)(n > 0 ? hi - lo : 0), (int)((a - lo) / sizeof(T))};
}

template <typename S>
struct TileGeom {
  int64_t r0, f0, e0;
  int nr, nf, ne;
};
template <typename S>
__device__ __forceinline__ TileGeom<S> tile_geom(const TileArgs<S>& A, int64_t t) {
  TileGeom<S> g;
  g.r0 = A.tile_row[t];
  g.f0 = A.tile_fib[t];
  g.e0 = A.tile_nz[t];
  g.nr = (int)(A.tile_row[t + 1] - g.r0);
  g.nf = (int)(A.tile_fib[t + 1] - g.f0);
  g.ne = (int)(A.tile_nz[t + 1] - g.e0);
  return g;
}

template <typename S>
struct View {
  const int64_t* rf;
  const uint32_t* fnz;
  const int32_t* fj;
  const uint32_t* k;
  const S* val;
  const uint8_t* aux;
  S* w;
  S* d;
  S* uj;
  uint16_t* frow;
};

// thread 0: bulk-copy the tile's slices into a stage
template <typename S, bool DO_R, int JAC>
__device__ __forceinline__ void tile_issue(const TileArgs<S>& A, const TileGeom<S>& g, unsigned char* st,
                                           uint64_t* bar) {
  using L = TileLayout<S, DO_R, JAC>;
  const Span a = span_of(A.row_fib + g.r0, g.nr + 1), b = span_of(A.fib_nz + g.f0, g.nf + 1),
             c = span_of(A.fib_j + g.f0, g.nf), d = span_of(A.nz_k + g.e0, g.ne),
             e = span_of(A.nz_val + g.e0, g.ne);
  Span f{nullptr, 0, 0};
  if (L::kP0) f = span_of(A.nz_aux + g.e0, g.ne);
  const uint64_t pol = policy_evict_first();
  mbar_expect_tx(bar, a.bytes + b.bytes + c.bytes + d.bytes + e.bytes + f.bytes);
  if (a.bytes) bulk_g2s(st + L::o_rf, a.src, a.bytes, bar, pol);
  if (b.bytes) bulk_g2s(st + L::o_fnz, b.src, b.bytes, bar, pol);
  if (c.bytes) bulk_g2s(st + L::o_fj, c.src, c.bytes, bar, pol);
  if (d.bytes) bulk_g2s(st + L::o_k, d.src, d.bytes, bar, pol);
  if (e.bytes) bulk_g2s(st + L::o_val, e.src, e.bytes, bar, pol);
  if (f.bytes) bulk_g2s(st + L::o_aux, f.src, f.bytes, bar, pol);
}

template <typename S, bool DO_R, int JAC>
__device__ __forceinline__ View<S> tile_view(const TileArgs<S>& A, const TileGeom<S>& g, unsigned char* st) {
  using L = TileLayout<S, DO_R, JAC>;
  View<S> v;
  v.rf = reinterpret_cast<const int64_t*>(st + L::o_rf) + span_of(A.row_fib + g.r0, 1).shift;
  v.fnz = reinterpret_cast<const uint32_t*>(st + L::o_fnz) + span_of(A.fib_nz + g.f0, 1).shift;
  v.fj = reinterpret_cast<const int32_t*>(st + L::o_fj) + span_of(A.fib_j + g.f0, 1).shift;
  v.k = reinterpret_cast<const uint32_t*>(st + L::o_k) + span_of(A.nz_k + g.e0, 1).shift;
  v.val = reinterpret_cast<const S*>(st + L::o_val) + span_of(A.nz_val + g.e0, 1).shift;
  v.aux = L::kP0 ? reinterpret_cast<const uint8_t*>(st + L::o_aux) + span_of(A.nz_aux + g.e0, 1).shift : nullptr;
  v.w = reinterpret_cast<S*>(st + L::o_w);
  v.d = reinterpret_cast<S*>(st + L::o_d);
  v.uj = reinterpret_cast<S*>(st + L::o_uj);
  v.frow = reinterpret_cast<uint16_t*>(st + L::o_frow);
  return v;
}

// all threads: async gathers of the tile's w_k (and D_u w, u_j) into its stage + fiber→row map
template <typename S, bool DO_R, int JAC>
__device__ __forceinline__ void tile_prepare(const TileArgs<S>& A, const TileGeom<S>& g, unsigned char* st) {
  using L = TileLayout<S, DO_R, JAC>;
  const int tid = threadIdx.x;
  const View<S> v = tile_view<S, DO_R, JAC>(A, g, st);
  for (int y = tid; y < g.ne; y += kThreads) {
    const uint32_t kr = v.k[y];
    const uint32_t k = kr & A.kmask;
    cp_async_s(v.w + y, A.w + k);
    if (L::kP0) {
      const uint32_t lc = (kr >> kKShift) & 3u;
      const S* cr = A.chain + (int64_t)k * A.d1;
      if (!A.packed) {
        cp_async_s(v.d + y, cr + lc);
      } else if ((int)lc + 1 < A.d1) {  // packed record: D_m at 1 + m
        cp_async_s(v.d + y, cr + 1 + lc);
      } else {  // D_d = −Σ_{m<d} D_m (a plain store; visible after the stage barrier)
        S sd = S(0);
        for (int m = 1; m < A.d1; ++m) sd = sd + __ldg(cr + m);
        v.d[y] = -sd;
      }
    }
  }
  if (L::kNeedU) {
    for (int x = tid; x < g.nf; x += kThreads) cp_async_s(v.uj + x, A.u + v.fj[x]);
  }
  cp_async_commit();
  if (L::kFrow) {
    for (int row = tid; row < g.nr; row += kThreads) {
      const int xa = (int)(v.rf[row] - g.f0), xb = (int)(v.rf[row + 1] - g.f0);
      for (int x = xa; x < xb; ++x) v.frow[x] = (uint16_t)row;
    }
  }
}

template <typename S, bool DO_R, int JAC>
__global__ void __launch_bounds__(kThreads) k_tile(const TileArgs<S> A) {
  using L = TileLayout<S, DO_R, JAC>;
  constexpr int NS = L::NS;
  constexpr int FPT = kTileFib / kThreads;  // fibers per thread
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::o_bar);
  S* fv = reinterpret_cast<S*>(smem + L::o_fv);
  S* bp = reinterpret_cast<S*>(smem + L::o_bp);
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  const int n_my = (A.n_tiles - (int)blockIdx.x + G - 1) / G;
  if (n_my <= 0) return;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < NS && q < n_my; ++q)
      tile_issue<S, DO_R, JAC>(A, tile_geom(A, (int64_t)blockIdx.x + (int64_t)q * G), smem + q * L::stage, &bars[q]);
  mbar_wait(&bars[0], 0);
  tile_prepare<S, DO_R, JAC>(A, tile_geom(A, (int64_t)blockIdx.x), smem);

  for (int q = 0; q < n_my; ++q) {
    const int s = q % NS;
    if (q + 1 < n_my) {
      const int s1 = (q + 1) % NS;
      mbar_wait(&bars[s1], ((q + 1) / NS) & 1);
      tile_prepare<S, DO_R, JAC>(A, tile_geom(A, (int64_t)blockIdx.x + (int64_t)(q + 1) * G), smem + s1 * L::stage);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();

    const TileGeom<S> g = tile_geom(A, (int64_t)blockIdx.x + (int64_t)q * G);
    const View<S> v = tile_view<S, DO_R, JAC>(A, g, smem + s * L::stage);
    // ---- phase B: fibers  a_f = Σ_k T_ijk w_k
    S areg[FPT];
#pragma unroll
    for (int c = 0; c < FPT; ++c) {
      const int x = tid + c * kThreads;
      areg[c] = S(0);
      if (x < g.nf) {
        const int ya = (int)(v.fnz[x] - (uint32_t)g.e0), yb = (int)(v.fnz[x + 1] - (uint32_t)g.e0);
        S a = S(0);
        for (int y = ya; y < yb; ++y) a += v.val[y] * v.w[y];
        areg[c] = a;
        S uj = S(0);
        if (L::kNeedU) uj = v.uj[x];
        if (DO_R) fv[x] = a * uj;
        if (JAC == kJacPicard) A.csr[g.f0 + x] = a;
        if (L::kP0) {
          // (T·₂u)_{iK} parts T_ijK u_j at (cell slot of K in row i, local index of j in K)
          const int row = v.frow[x];
          const int rowbase = (int)(v.fnz[v.rf[row] - g.f0] - (uint32_t)g.e0);
          for (int y = ya; y < yb; ++y)
            bp[rowbase + (int)v.aux[y] * A.d1 + (int)((v.k[y] >> kKShift) & 3u)] = v.val[y] * uj;
        }
      }
    }
    if (DO_R || L::kP0) __syncthreads();
    if (L::kP0) {
      // B_iK = Σ_m (T_{i v_m K} u_{v_m}) once per (row, cell) of the tile, compacted in place to
      // bp[cell]: rows of P0-W tensors hold d+1 nonzeros per cell, so cell c's parts sit at
      // bp[c·(d+1) .. +d] (fixed summation order m = 0..d)
      constexpr int CPT = (kTileNnz / 2 + kThreads - 1) / kThreads;  // cells per thread (d+1 >= 2)
      S bs[CPT];
      const int ncell = g.ne / A.d1;
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int cc = tid + c * kThreads;
        S B = S(0);
        if (cc < ncell)
          for (int m = 0; m < A.d1; ++m) B += bp[cc * A.d1 + m];
        bs[c] = B;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < CPT; ++c)
        if (tid + c * kThreads < ncell) bp[tid + c * kThreads] = bs[c];
      __syncthreads();
    }
    // ---- phase C: rows and Newton terms
    if (DO_R) {
      for (int row = tid; row < g.nr; row += kThreads) {
        const int xa = (int)(v.rf[row] - g.f0), xb = (int)(v.rf[row + 1] - g.f0);
        S acc = S(0);
        for (int x = xa; x < xb; ++x) acc += fv[x];
        A.r[g.r0 + row] = acc;
      }
    }
    if (L::kWV) {
      // J_(i,m) = A_(i,m) + c_m Σ_{(j, k=m) in row i} T_ijm u_j,  c_m = 1 or 2u_m (SQUARE)
#pragma unroll
      for (int c = 0; c < FPT; ++c) {
        const int x = tid + c * kThreads;
        if (x < g.nf) {
          const int row = v.frow[x];
          const uint32_t m = (uint32_t)v.fj[x];
          const int xa = (int)(v.rf[row] - g.f0), xb = (int)(v.rf[row + 1] - g.f0);
          S acc = S(0);
          for (int x2 = xa; x2 < xb; ++x2) {
            const S uj = v.uj[x2];
            const int ya = (int)(v.fnz[x2] - (uint32_t)g.e0), yb = (int)(v.fnz[x2 + 1] - (uint32_t)g.e0);
            for (int y = ya; y < yb; ++y)
              if ((v.k[y] & A.kmask) == m) acc += v.val[y] * uj;
          }
          const S um = A.dmode ? ld_ro(A.u + m) : S(0);
          S cm = S(1);
          if (A.dmode == 1) cm = S(2) * um;
          if (A.dmode == 2) {
            const S iv = S(1) / (S(A.pk) + um);
            cm = -(iv * iv);
          }
          A.csr[g.f0 + x] = areg[c] + cm * acc;
        }
      }
    }
    if (L::kP0) {
      // J_ij = A_ij + Σ_{K in fiber} B_{iK} (D_u w)_{K, loc(j)}
#pragma unroll
      for (int c = 0; c < FPT; ++c) {
        const int x = tid + c * kThreads;
        if (x < g.nf) {
          const int row = v.frow[x];
          const int rowbase = (int)(v.fnz[v.rf[row] - g.f0] - (uint32_t)g.e0);
          const int ya = (int)(v.fnz[x] - (uint32_t)g.e0), yb = (int)(v.fnz[x + 1] - (uint32_t)g.e0);
          S acc = areg[c];
          const int cbase = rowbase / A.d1;
          for (int y = ya; y < yb; ++y) acc += bp[cbase + (int)v.aux[y]] * v.d[y];
          A.csr[g.f0 + x] = acc;
        }
      }
    }
    __syncthreads();
    if (tid == 0 && q + NS < n_my)
      tile_issue<S, DO_R, JAC>(A, tile_geom(A, (int64_t)blockIdx.x + (int64_t)(q + NS) * G), smem + s * L::stage,
                               &bars[s]);
  }
}

int g_num_sms[64] = {0};

template <typename S, bool DO_R, int JAC>
egfem_status run_tile(const egfem_tensor* t, const TileArgs<S>& A, cudaStream_t s) {
  using L = TileLayout<S, DO_R, JAC>;
  if (t->n_tiles <= 0) return EGFEM_OK;
  auto fn = k_tile<S, DO_R, JAC>;
  EGFEM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, L::bytes));
  int dev = t->device;
  if (g_num_sms[dev & 63] == 0) {
    int n = 0;
    EGFEM_CUDA_TRY(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    g_num_sms[dev & 63] = n;
  }
  int per_sm = 0;
  EGFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, L::bytes));
  const int grid = std::max(1, std::min(t->n_tiles, std::max(per_sm, 1) * g_num_sms[dev & 63]));
  fn<<<grid, kThreads, L::bytes, s>>>(A);
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

template <typename S>
egfem_status tile_dispatch(const egfem_tensor* t, bool do_r, int jac, egfem_interp_kind kind, double p, const void* u,
                           const void* w, const void* chain, void* r, void* csr, cudaStream_t s) {
  TileArgs<S> A;
  A.tile_row = t->tile_row;
  A.tile_fib = t->tile_fib;
  A.tile_nz = t->tile_nz;
  A.n_tiles = t->n_tiles;
  A.row_fib = t->row_fib;
  A.fib_j = t->fib_j;
  A.fib_nz = t->fib_nz;
  A.nz_k = t->nz_k;
  A.nz_val = static_cast<const S*>(t->nz_val);
  A.nz_aux = t->nz_aux;
  A.u = static_cast<const S*>(u);
  A.w = static_cast<const S*>(w);
  A.chain = static_cast<const S*>(chain);
  A.r = static_cast<S*>(r);
  A.csr = static_cast<S*>(csr);
  A.d1 = t->dim + 1;
  A.packed = jac == kJacNewtonP0 && packed_chain_kind(kind);
  A.dmode = kind == EGFEM_INTERP_SQUARE ? 1 : (kind == EGFEM_INTERP_RECIPROCAL ? 2 : 0);
  A.pk = p;
  A.kmask = t->kmask();
  if (do_r) {
    switch (jac) {
      case kJacNone: return run_tile<S, true, kJacNone>(t, A, s);
      case kJacPicard: return run_tile<S, true, kJacPicard>(t, A, s);
      case kJacNewtonWV: return run_tile<S, true, kJacNewtonWV>(t, A, s);
      default: return run_tile<S, true, kJacNewtonP0>(t, A, s);
    }
  }
  switch (jac) {
    case kJacPicard: return run_tile<S, false, kJacPicard>(t, A, s);
    case kJacNewtonWV: return run_tile<S, false, kJacNewtonWV>(t, A, s);
    case kJacNewtonP0: return run_tile<S, false, kJacNewtonP0>(t, A, s);
    default: return EGFEM_ERR_INVALID_ARGUMENT;
  }
}

// ------------------------------------------------------------------ batched apply
// One CTA per tile; the tile's (k, value) and fiber structure are staged in shared
// memory once and reused by all B pairs.  Warp w handles pairs [32w', 32w'+32) in
// chunks; lane = pair.  NODE_MAJOR vectors make every gather a coalesced 256 B row.
template <typename S, bool NODE_MAJOR>
__global__ void __launch_bounds__(kThreads) k_batched(const int64_t* __restrict__ tile_row,
                                                      const int64_t* __restrict__ row_fib,
                                                      const int32_t* __restrict__ fib_j,
                                                      const uint32_t* __restrict__ fib_nz,
                                                      const uint32_t* __restrict__ nz_k, const S* __restrict__ nz_val,
                                                      bool p0, int32_t B, int64_t n_u, int64_t n_f,
                                                      const S* __restrict__ U, const S* __restrict__ W,
                                                      S* __restrict__ R) {
  __shared__ S s_val[kTileNnz];
  __shared__ uint32_t s_k[kTileNnz];
  __shared__ int32_t s_fnz[kTileFib + 1];
  __shared__ int32_t s_fj[kTileFib];
  __shared__ int32_t s_rf[kTileRows + 1];
  const int tid = threadIdx.x;
  const int64_t r0 = tile_row[blockIdx.x], r1 = tile_row[blockIdx.x + 1];
  const int nr = (int)(r1 - r0);
  const int64_t f0 = row_fib[r0];
  const int nf = (int)(row_fib[r1] - f0);
  const uint32_t e0 = fib_nz[f0];
  const int ne = (int)(fib_nz[f0 + nf] - e0);
  for (int e = tid; e < ne; e += kThreads) {
    const uint32_t kk = ld_stream(nz_k + e0 + e);
    s_k[e] = kk & (p0 ? kKMask : kKMaskAny);
    s_val[e] = ld_stream(nz_val + e0 + e);
  }
  for (int x = tid; x <= nf; x += kThreads) s_fnz[x] = (int32_t)(fib_nz[f0 + x] - e0);
  for (int x = tid; x < nf; x += kThreads) s_fj[x] = fib_j[f0 + x];
  for (int x = tid; x <= nr; x += kThreads) s_rf[x] = (int32_t)(row_fib[r0 + x] - f0);
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int nchunks = (B + 31) / 32;
  for (int task = warp; task < nchunks * nr; task += kThreads / 32) {
    const int chunk = task % nchunks, row = task / nchunks;
    const int p = chunk * 32 + lane;
    if (p >= B) continue;
    S acc = S(0);
    for (int x = s_rf[row]; x < s_rf[row + 1]; ++x) {
      S a = S(0);
      for (int y = s_fnz[x]; y < s_fnz[x + 1]; ++y) {
        const int64_t k = s_k[y];
        const S wv = NODE_MAJOR ? ld_ro(W + k * B + p) : ld_ro(W + (int64_t)p * n_f + k);
        a += s_val[y] * wv;
      }
      const int64_t j = s_fj[x];
      const S uv = NODE_MAJOR ? ld_ro(U + j * B + p) : ld_ro(U + (int64_t)p * n_u + j);
      acc += a * uv;
    }
    if (NODE_MAJOR)
      R[(r0 + row) * B + p] = acc;
    else
      R[(int64_t)p * n_u + r0 + row] = acc;
  }
}

template <typename S>
__global__ void k_halo(const int32_t* __restrict__ idx, int64_t n, const S* __restrict__ src, S* __restrict__ dst,
                       bool pack) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  if (pack)
    dst[q] = src[idx[q]];
  else
    dst[idx[q]] = src[q];
}

}  // namespace

// Interp work items: W DOFs for the pointwise kinds on W = V, mesh cells otherwise.
static bool interp_pointwise_wv(const egfem_tensor* t, egfem_interp_kind kind) {
  return kind == EGFEM_INTERP_IDENTITY || (kind == EGFEM_INTERP_SQUARE && t->w_is_v) ||
         (kind == EGFEM_INTERP_RECIPROCAL && t->w_is_v);
}
int64_t interp_items(const egfem_tensor* t, egfem_interp_kind kind) {
  return interp_pointwise_wv(t, kind) ? t->n_f : t->n_cells;
}

// Items [lo, hi) of the work: every kernel runs on base pointers shifted to item lo (cell
// records, V/W DOF tables, and for the IOTA / copy kernels w and chain), so a sub-range is
// the same per-item arithmetic as the whole call.
egfem_status launch_interp(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u, void* w,
                           void* chain, int64_t lo, int64_t hi, cudaStream_t s) {
  const bool f64 = t->dtype == EGFEM_F64;
  const size_t vs = f64 ? 8 : 4;
  const int64_t n = hi - lo;
  if (n <= 0) return EGFEM_OK;
  if (interp_pointwise_wv(t, kind)) {
    const int grid = std::max(1, std::min(nblk(n), 148 * 16));
    const int mode = kind == EGFEM_INTERP_IDENTITY ? 0 : (kind == EGFEM_INTERP_SQUARE ? 1 : 2);
    const void* ul = (const char*)u + vs * lo;
    void* wl = (char*)w + vs * lo;
    if (f64)
      k_interp_copy<double><<<grid, 256, 0, s>>>((const double*)ul, (double*)wl, n, mode, p);
    else
      k_interp_copy<float><<<grid, 256, 0, s>>>((const float*)ul, (float*)wl, n, mode, p);
    count_launch();
  } else if (kind == EGFEM_INTERP_RECIPROCAL || kind == EGFEM_INTERP_SQUARE) {  // cell-wise W, V = P1
    const int mode = kind == EGFEM_INTERP_RECIPROCAL ? 0 : 1;
    const int d1 = t->dim + 1;
    const int32_t* vd = t->vdofs + lo * d1;
    const int32_t* wd = t->wdofs + lo * t->nwc;
    if (t->wdofs_is_iota) {  // outputs of cells [lo, hi) are the spans from W DOF lo·nw on
      const int sm = 128 * t->nwc * (1 + d1) * (int)vs;
      const int64_t wo = lo * t->nwc;
      if (f64) {
        if (sm > 48 * 1024)
          EGFEM_CUDA_TRY(cudaFuncSetAttribute(k_interp_points_blk<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        k_interp_points_blk<double><<<nblk(n, 128), 128, sm, s>>>(vd, t->wpts, n, d1, t->nwc, (const double*)u,
                                                                  (double*)w + wo,
                                                                  chain ? (double*)chain + wo * d1 : nullptr, mode, p);
      } else {
        if (sm > 48 * 1024)
          EGFEM_CUDA_TRY(cudaFuncSetAttribute(k_interp_points_blk<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        k_interp_points_blk<float><<<nblk(n, 128), 128, sm, s>>>(vd, t->wpts, n, d1, t->nwc, (const float*)u,
                                                                 (float*)w + wo,
                                                                 chain ? (float*)chain + wo * d1 : nullptr, mode, p);
      }
    } else if (f64) {
      k_interp_points<double><<<nblk(n, 128), 128, 0, s>>>(vd, wd, t->wpts, n, d1, t->nwc, (const double*)u,
                                                           (double*)w, (double*)chain, mode, p);
    } else {
      k_interp_points<float><<<nblk(n, 128), 128, 0, s>>>(vd, wd, t->wpts, n, d1, t->nwc, (const float*)u,
                                                          (float*)w, (float*)chain, mode, p);
    }
    count_launch();
  } else if (kind == EGFEM_INTERP_GRADPOW_P0 || kind == EGFEM_INTERP_MINSURF_P0) {
    const int grid = std::max(1, nblk(n, 128));  // capped at one resident wave below
    const int d1 = t->dim + 1;
    const int32_t* cl = t->cells + lo * d1;
    const int32_t* vd = t->vdofs + lo * t->nV;
    const int32_t* wd = t->wdofs + lo * t->nwc;
#define EGFEM_GP4(S, D, SA, IO, CF)                                                                   \
  do {                                                                                                \
    int per_sm = 0;                                                                                   \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_interp_gradpow<S, D, SA, IO, CF>, 128, 0); \
    const int g = (int)std::min<int64_t>(grid, (int64_t)std::max(per_sm, 1) * 148);                   \
    S* wl = (IO && w) ? (S*)w + lo : (S*)w; /* w may be NULL (packed kinds) */                        \
    S* cl2 = (IO && chain) ? (S*)chain + lo * (D + 1) : (S*)chain;                                    \
    k_interp_gradpow<S, D, SA, IO, CF><<<g, 128, 0, s>>>(D == 3 ? t->coords4 : t->coords, t->coordsf, cl, vd, \
                                                         wd, n, (const S*)u, wl, cl2, p,              \
                                                         kind == EGFEM_INTERP_MINSURF_P0, t->nwc);     \
  } while (0)
#define EGFEM_GP3(S, D, SA, IO)                                                 \
  do {                                                                          \
    if (D >= 2 && t->coordsf) EGFEM_GP4(S, D, SA, IO, true);                    \
    else EGFEM_GP4(S, D, SA, IO, false);                                        \
  } while (0)
#define EGFEM_GP(S, D)                                                          \
  do {                                                                          \
    if (geo_interp_ok(t) && D == 3) {                                              \
      int per_sm = 0;                                                                                   \
      auto kg = sizeof(S) == 8 ? k_interp_gradpow_geo6<S, true> : k_interp_gradpow_geo<S, true>;        \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kg, 128, 0);                               \
      const int g = (int)std::min<int64_t>(grid, (int64_t)std::max(per_sm, 1) * 148);                   \
      kg<<<g, 128, 0, s>>>(t->gtab, t->n_geo, t->gcls + lo, cl, n, (const S*)u,    \
                                                w ? (S*)w + lo : (S*)w,                                 \
                                                chain ? (S*)chain + lo * 4 : (S*)chain, p,              \
                                                kind == EGFEM_INTERP_MINSURF_P0);                       \
    } else if (t->vdofs_is_cells && t->wdofs_is_iota && t->nwc == 1) EGFEM_GP3(S, D, true, true);       \
    else EGFEM_GP3(S, D, false, false);                                         \
  } while (0)
    if (f64) {
      if (t->dim == 1) EGFEM_GP(double, 1); else if (t->dim == 2) EGFEM_GP(double, 2); else EGFEM_GP(double, 3);
    } else {
      if (t->dim == 1) EGFEM_GP(float, 1); else if (t->dim == 2) EGFEM_GP(float, 2); else EGFEM_GP(float, 3);
    }
#undef EGFEM_GP4
#undef EGFEM_GP3
#undef EGFEM_GP
    count_launch();
  } else {
    const int32_t* vd = t->vdofs + lo * 3;
    const int32_t* wd = t->wdofs + lo * 6;
    if (f64)
      k_interp_p1p2sq<double><<<nblk(n), 256, 0, s>>>(vd, wd, n, (const double*)u, (double*)w);
    else
      k_interp_p1p2sq<float><<<nblk(n), 256, 0, s>>>(vd, wd, n, (const float*)u, (float*)w);
    count_launch();
  }
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

egfem_status launch_tile(const egfem_tensor* t, bool do_r, int jac, egfem_interp_kind kind, double p, const void* u,
                         const void* w, const void* chain, void* r, void* csr_vals, cudaStream_t s) {
  // Row-group kernels (egfem_rows.cu) unless a row is too long or EGFEM_PATH=tile forces the
  // TMA-pipelined tile kernel (kept as the general path and as a cross-check in the tests).
  // EGFEM_PATH=rows skips the cell-major P0 kernel (egfem_cells.cu) for the row kernel.
  static const char* force = getenv("EGFEM_PATH");
  const bool tile = force && force[0] == 't';
  const bool rows_only = force && force[0] == 'r';
  if (!tile && !rows_only && cells_path_ok(t, jac))
    return launch_cells(t, do_r, jac, jac == 3 && packed_chain_kind(kind), u, w, chain, r, csr_vals, s);
  if (!tile && !rows_only && dense1_path_ok(t, jac))
    return launch_dense1(t, 0, t->n_u, do_r, jac, kind, p, u, w, r, csr_vals, s);
  if (!tile && rows_path_ok(t, jac)) return launch_rows(t, do_r, jac, kind, p, u, w, chain, r, csr_vals, s);
  if (t->dtype == EGFEM_F64) return tile_dispatch<double>(t, do_r, jac, kind, p, u, w, chain, r, csr_vals, s);
  return tile_dispatch<float>(t, do_r, jac, kind, p, u, w, chain, r, csr_vals, s);
}

std::string dispatch_name(const egfem_tensor* t, int entry, int jac) {
  if (entry == 3) {
    static const char* forceb = getenv("EGFEM_BATCHED");
    const bool fc = forceb && forceb[0] == 'c', fd = forceb && forceb[0] == 'd';
    if (group_path_ok(t, EGFEM_LAYOUT_NODE_MAJOR) && !fc && !fd)
      return std::string("egfem_grp_* (compiled row groups, egfem_group.cu)") + group_plan_info(t);
    if (dense_path_ok(t) && !fc) return "k_dense (per-row dense blocks, egfem_dense.cu)";
    return "k_batched (CSF tiles, egfem_kernels.cu)";
  }
  static const char* force = getenv("EGFEM_PATH");
  const bool tile = force && force[0] == 't';
  const bool rows_only = force && force[0] == 'r';
  if (!tile && !rows_only && cells_path_ok(t, jac))
    return std::string("k_cell (cell-major P0, egfem_cells.cu; ") + cells_variant(t) + ")";
  if (!tile && !rows_only && dense1_path_ok(t, jac)) return "k_dense1 (dense single-vector W = V, egfem_dense.cu)";
  if (!tile && rows_path_ok(t, jac)) return "k_seg (row groups on the CSF, egfem_rows.cu)";
  return "k_tile (TMA row tiles, egfem_kernels.cu)";
}

// Rows [lo, hi): a shallow view of the tensor whose row arrays start at row lo (row_nz,
// row_fib hold absolute nonzero / fiber offsets, so the streams, csr and the fiber data are
// addressed as in the whole call) and whose diagonal offset moves with it; r is shifted.
// Only the row-group kernels (cell-major, segmented) take a view.
egfem_status launch_tile_rows(const egfem_tensor* t, int64_t lo, int64_t hi, bool do_r, int jac,
                              egfem_interp_kind kind, double p, const void* u, const void* w, const void* chain,
                              void* r, void* csr_vals, cudaStream_t s) {
  if (lo == 0 && hi == t->n_u) return launch_tile(t, do_r, jac, kind, p, u, w, chain, r, csr_vals, s);
  if (hi <= lo) return EGFEM_OK;
  static const char* force = getenv("EGFEM_PATH");
  const bool tile = force && force[0] == 't';
  const bool rows_only = force && force[0] == 'r';
  const bool cells = !tile && !rows_only && cells_path_ok(t, jac);
  if (!cells && !tile && !rows_only && dense1_path_ok(t, jac))  // rows [lo, hi) of the row-order dense kernel
    return launch_dense1(t, lo, hi, do_r, jac, kind, p, u, w, r, csr_vals, s);
  if (!cells && (tile || !rows_path_ok(t, jac))) {
    set_error("row sub-ranges need a row-group kernel (rows of at most 256 nonzeros)");
    return EGFEM_ERR_UNSUPPORTED;
  }
  egfem_tensor v;
  v.device = t->device;
  v.dtype = t->dtype;
  v.has_mesh = t->has_mesh;
  v.dim = t->dim;
  v.n_u = hi - lo;
  v.n_f = t->n_f;
  v.vfam = t->vfam;
  v.wfam = t->wfam;
  v.form = t->form;
  v.nnz = t->nnz;
  v.n_fib = t->n_fib;
  v.w_is_v = t->w_is_v;
  v.w_p0 = t->w_p0;
  v.nwc = t->nwc;
  v.newton_wv_ok = t->newton_wv_ok;
  v.max_row_nnz = t->max_row_nnz;
  v.max_row_fib = t->max_row_fib;
  v.row_fib = t->row_fib + lo;
  v.row_nz = t->row_nz + lo;
  v.fib_j = t->fib_j;
  v.fib_nz = t->fib_nz;
  v.nz_k = t->nz_k;
  v.nz_val = t->nz_val;
  v.nz_aux = t->nz_aux;
  v.nz_kpos = t->nz_kpos;
  v.fib_kr = t->fib_kr;
  v.ck_k = t->ck_k;
  v.ck_val = t->ck_val;
  v.ck_b = t->ck_b;
  v.ck_m = t->ck_m;
  v.ck_kb = t->ck_kb ? t->ck_kb + lo : nullptr;
  v.ck_fb = t->ck_fb;
  v.ck_pb = t->ck_pb;
  v.ck_ks = t->ck_ks;
  v.row_begin = t->row_begin + lo;
  v.col_begin = t->col_begin;
  void* rl = r ? (char*)r + (t->dtype == EGFEM_F64 ? 8 : 4) * lo : nullptr;
  if (cells) return launch_cells(&v, do_r, jac, jac == 3 && packed_chain_kind(kind), u, w, chain, rl, csr_vals, s);
  return launch_rows(&v, do_r, jac, kind, p, u, w, chain, rl, csr_vals, s);
}

egfem_status launch_batched(const egfem_tensor* t, int32_t batch, egfem_layout layout, const void* U, const void* W,
                            void* R, cudaStream_t s) {
  if (t->n_tiles == 0) return EGFEM_OK;
  // dense-local-block kernel (egfem_dense.cu) for W = V stencils; EGFEM_BATCHED=csf forces
  // the CSF tile kernel below
  static const char* force = getenv("EGFEM_BATCHED");
  // compiled row-group kernels (egfem_group.cu) first; EGFEM_BATCHED=dense forces the per-row
  // dense-block kernel
  if (group_path_ok(t, layout) && !(force && (force[0] == 'c' || force[0] == 'd')))
    return launch_groups(t, batch, U, W, R, s);
  if (dense_path_ok(t) && !(force && force[0] == 'c')) return launch_dense(t, batch, layout, U, W, R, s);
  const bool p0 = t->has_mesh && t->w_p0;
  const bool nm = layout == EGFEM_LAYOUT_NODE_MAJOR;
#define EGFEM_B(S, NM)                                                                                           \
  k_batched<S, NM><<<t->n_tiles, kThreads, 0, s>>>(t->tile_row, t->row_fib, t->fib_j, t->fib_nz, t->nz_k,        \
                                                   (const S*)t->nz_val, p0, batch, t->n_u, t->n_f, (const S*)U,  \
                                                   (const S*)W, (S*)R)
  if (t->dtype == EGFEM_F64) {
    if (nm) EGFEM_B(double, true); else EGFEM_B(double, false);
  } else {
    if (nm) EGFEM_B(float, true); else EGFEM_B(float, false);
  }
#undef EGFEM_B
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

egfem_status launch_halo(const egfem_tensor* t, const int32_t* idx, int64_t n, const void* src, void* dst, bool pack,
                         cudaStream_t s) {
  if (n <= 0) return EGFEM_OK;
  if (t->dtype == EGFEM_F64)
    k_halo<double><<<nblk(n), 256, 0, s>>>(idx, n, (const double*)src, (double*)dst, pack);
  else
    k_halo<float><<<nblk(n), 256, 0, s>>>(idx, n, (const float*)src, (float*)dst, pack);
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

}  // namespace egfem

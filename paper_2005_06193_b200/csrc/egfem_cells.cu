// Cell-major row kernel of libegfem.so (B200 / sm_100a) for P0 W: steps (2)+(3) of the
// p-Laplace-type forms T_ijK = ∫_K ψ_K ∇φ_i·∇φ_j (§5.5).
//
// With W = P0 every nonzero of row i belongs to exactly one cell K ∋ i, and the cell
// contributes one nonzero (i, v_m, K) for each of its d+1 vertices v_m.  Besides the
// canonical (i, j, k) CSF the builder keeps the same nonzeros in the mode order
// i -> K -> m ("cell-major"): per row, its cells in ascending K, each with the d+1 values
// T_{i v_m K} in local-vertex order m.  In that order the Newton chain factor
//   B_iK = (T·₂u)_{iK} = Σ_m T_{i v_m K} u_{v_m}
// is an in-register sum over one lane's cell, the residual is
//   r_i  = Σ_K w_K B_iK
// with one w gather per cell, and the Jacobian terms
//   t_{i v_m K} = T_{i v_m K} w_K [+ B_iK (D_u w)_{K m}]
// go either to the diagonal fiber (i, i) — one nonzero per cell, summed in registers and
// reduced by a butterfly — or, scattered once into the row's canonical positions, to the short
// off-diagonal fibers, which the lane owning the fiber sums in canonical order.  Per nonzero the stream carries the value
// and a 16-bit (fiber, canonical position) pair; per cell the 32-bit K.
//
// Layout per row group (G lanes, CPL cells per lane — lane l takes cells l, l+G, l+2G, so one
// warp-wide gather touches a few neighbouring cells' lines — grid-stride rows): the next row's
// (K, value, fiber|pos) slices are fetched into a second shared-memory stage while the current
// row is reduced, by 16-byte cp.async.cg (L2 evict-first) or, when a warp holds >= 8 rows,
// by three TMA bulk copies per warp (its rows are consecutive) completing on an mbarrier.  Every sum
// runs in a fixed order: bitwise reproducible; fused and separate launches agree bitwise.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "egfem_internal.cuh"
#include "egfem_interp.cuh"

namespace egfem {
namespace {

// kJacNewtonPK: P0 Newton with the packed chain of the gradient kinds (include/egfem.h
// egfem_interp: [w_K, ∂w/∂u_0 .. ∂w/∂u_{d−1}], ∂w/∂u_d = −Σ: one gather per cell)
enum { kJacNone = 0, kJacPicard = 1, kJacNewtonP0 = 3, kJacNewtonPK = 4 };
// threads per CTA: 256 for the fp64 Newton / apply kernels (2-3 CTAs/SM), 128 for fp32 and for
// the fp64 Picard matrix (measured on cfg4: fp32 fused 0.51 -> 0.47 ms, fp64 Picard 0.51 ->
// 0.48 ms; fp64 fused is faster with 256)
template <typename S, int JAC>
__host__ __device__ constexpr int cell_threads() {
  return (sizeof(S) == 4 || JAC == kJacPicard) ? 128 : 256;
}

template <typename S>
struct CellArgs {
  int64_t n_u;
  const int64_t* row_nz;   // first canonical nonzero of each row (= (d+1) x first cell)
  const int64_t* row_fib;  // first fiber (CSR slot) of each row
  const int32_t* fib_j;
  const uint32_t* fib_nz;
  const uint32_t* ck_k;    // per cell of a row: K
  const S* ck_val;         // per nonzero, cell-major: T_{i v_m K}
  const uint16_t* ck_b;    // per nonzero: fiber index in row (low byte) | canonical position (high)
  const uint64_t* ck_m = nullptr;   // per cell of a row: the packed word (egfem_tensor::ck_m), PM kernels
  const uint32_t* ck_kb = nullptr;  // per row: K of its first cell (PM)
  int fb = 0, fw = 0, ks = 0;       // PM field widths: fiber bits, fiber + position bits, shift of K − kb
  const S* u;
  const S* w;
  const S* chain;          // (D_u w)_{K m}, N_f x (d+1)
  S* r;
  S* csr;
  int64_t diag_off;        // column of row i's diagonal = i + diag_off (local tensors of a partition)
  bool chain32;            // chain is 32-byte aligned (one 256-bit load per cell row)
  int pf;                  // apply-only kernel: prefetch the value span of the warp's rows 2 steps ahead
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// TMA 1D bulk copies completing on an mbarrier (one lane per warp issues them)
__device__ __forceinline__ void bar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
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
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// 16-byte-aligned span around [p, p+n): start, byte count; returns the element shift
template <typename T>
__device__ __forceinline__ int span16(const T* p, int n, const char** lo_out, uint32_t* bytes) {
  const uint64_t a = reinterpret_cast<uint64_t>(p);
  const uint64_t lo = a & ~uint64_t(15);
  *bytes = n > 0 ? (uint32_t)(((a + (uint64_t)n * sizeof(T) + 15) & ~uint64_t(15)) - lo) : 0u;
  *lo_out = reinterpret_cast<const char*>(lo);
  return (int)((a - lo) / sizeof(T));
}
__device__ __forceinline__ void wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// 16-byte async copies of the span around [p, p+n) to shared address dst; returns the shift.
template <typename T, int G, int CAP>
__device__ __forceinline__ int stage_span(uint32_t dst, const T* p, int n, int lane, uint64_t pol) {
  constexpr int IT = ((CAP * (int)sizeof(T) + 31) / 16 + G - 1) / G;
  const uint64_t a = reinterpret_cast<uint64_t>(p);
  const uint64_t lo = a & ~uint64_t(15);
  const int chunks = n > 0 ? (int)((((a + (uint64_t)n * sizeof(T) + 15) & ~uint64_t(15)) - lo) >> 4) : 0;
  const char* src = reinterpret_cast<const char*>(lo) + 16 * lane;
  dst += 16 * lane;
#pragma unroll
  for (int it = 0; it < IT; ++it)
    if (lane + it * G < chunks) cp16(dst + 16 * G * it, src + 16 * G * it, pol);
  return (int)((a - lo) / sizeof(T));
}

__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float xmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float xadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double xfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float xfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// Shared memory per row group: two stages of (K, value, fiber|pos) slices and the Jacobian
// scratch.  With warp-level bulk staging the 32/G groups of a warp pool their stage regions
// into one warp stage per buffer (the warp's rows are consecutive, so their slices are one
// contiguous span per array) and the warp's two mbarriers sit in group 0's tail.
template <typename S, int D1, int G, int CPL, bool JT, int SUN = 0, bool NS = false>
struct CellSmem {
  static constexpr int CC = G * CPL;  // cells per row (max)
  static constexpr int CE = CC * D1;  // nonzeros per row (max)
  // each slice gets 32 B of slack (its 16-byte-aligned span may start up to 15 B early and
  // end up to 15 B late) and starts 16-byte aligned (cp.async destination)
  // (per-lane cp.async path: K and the (fiber, position) pairs only — the values go straight
  // to registers, so st_v is an empty slot)
  static constexpr int st_k = 0;
  static constexpr int st_v = (st_k + CC * 4 + 32 + 15) & ~15;
  static constexpr int st_b = st_v;
  static constexpr int stage = NS ? 0 : (st_b + CE * 2 + 32 + 15) & ~15;
  static constexpr int o_t = 2 * stage;  // S[CE]: Jacobian terms at canonical positions
  // warp stage (bulk): WPG groups' slices back to back, each array with 32 B of slack
  static constexpr int WPG = 32 / G;
  static constexpr int w_k = 0;
  static constexpr int w_v = (w_k + WPG * CC * 4 + 32 + 15) & ~15;
  static constexpr int w_b = (w_v + WPG * CE * (int)sizeof(S) + 32 + 15) & ~15;
  static constexpr int wstage = (w_b + WPG * CE * 2 + 32 + 15) & ~15;
  static constexpr int o_u = (o_t + (JT ? CE * (int)sizeof(S) : 0) + 15) & ~15;  // s_t only with a Jacobian
  static constexpr int raw = (o_u + SUN * (int)sizeof(S) + 15) & ~15;              // s_u: u at the row's fibers
  // per-warp layout for bulk staging: [2 warp stages][WPG x s_t][2 mbarriers]
  static constexpr int wo_t = 2 * wstage;
  static constexpr int wo_u = (wo_t + (JT ? WPG * CE * (int)sizeof(S) : 0) + 15) & ~15;
  static constexpr int wo_bar = (wo_u + WPG * SUN * (int)sizeof(S) + 15) & ~15;
  static constexpr int wraw = wo_bar + 16;
  static constexpr int wbytes = wraw + ((16 - wraw % 128) + 128) % 128;
  // group stride = 16 (mod 128): the groups of a warp start on different bank quads, so
  // their same-offset accesses do not collide
  static constexpr int bytes = raw + ((16 - raw % 128) + 128) % 128;
};

// the D1 values of one cell (16-byte vector loads when the cell is 16-byte aligned)
template <typename S, int D1>
__device__ __forceinline__ void load_cell(const S* p, bool vec, S* out) {
  if constexpr ((D1 * sizeof(S)) % 16 == 0) {
    if (vec) {
      constexpr int NV = D1 * (int)sizeof(S) / 16;
      constexpr int PER = 16 / (int)sizeof(S);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if constexpr (sizeof(S) == 8) {
          const double2 x = reinterpret_cast<const double2*>(p)[v];
          out[v * PER] = x.x;
          out[v * PER + 1] = x.y;
        } else {
          const float4 x = reinterpret_cast<const float4*>(p)[v];
          out[v * PER] = x.x;
          out[v * PER + 1] = x.y;
          out[v * PER + 2] = x.z;
          out[v * PER + 3] = x.w;
        }
      }
      return;
    }
  }
#pragma unroll
  for (int m = 0; m < D1; ++m) out[m] = p[m];
}
// the D1 values of one cell from global memory (16-byte read-only vector loads; D1·sizeof(S) % 16 == 0)
template <typename S, int D1>
__device__ __forceinline__ void load_cell_ldg(const S* p, S* out, bool a32 = false) {
  if constexpr (sizeof(S) == 8 && D1 == 4) {
    if (a32) {  // 32-byte aligned: one 256-bit load
      asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(out[0]), "=d"(out[1]), "=d"(out[2]), "=d"(out[3]) : "l"(p));
      return;
    }
  }
  constexpr int NV = D1 * (int)sizeof(S) / 16;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if constexpr (sizeof(S) == 8) {
      const double2 x = __ldg(reinterpret_cast<const double2*>(p) + v);
      out[2 * v] = x.x;
      out[2 * v + 1] = x.y;
    } else {
      const float4 x = __ldg(reinterpret_cast<const float4*>(p) + v);
      out[4 * v] = x.x;
      out[4 * v + 1] = x.y;
      out[4 * v + 2] = x.z;
      out[4 * v + 3] = x.w;
    }
  }
}
// the same through L2 only (data written earlier in the same launch by another SM)
template <typename S, int D1>
__device__ __forceinline__ void load_cell_cg(const S* p, S* out, bool a32 = false) {
  if constexpr (sizeof(S) == 8 && D1 == 4) {
    if (a32) {
      // address dependent on shared-memory data read after the launch's acquire: never hoisted
      asm("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(out[0]), "=d"(out[1]), "=d"(out[2]), "=d"(out[3]) : "l"(p));
      return;
    }
  }
  if constexpr (sizeof(S) == 4 && D1 == 4) {  // one 16-byte load (the chain rows are 16-byte aligned)
    const float4 x = __ldcg(reinterpret_cast<const float4*>(p));
    out[0] = x.x;
    out[1] = x.y;
    out[2] = x.z;
    out[3] = x.w;
    return;
  }
#pragma unroll
  for (int m = 0; m < D1; ++m) out[m] = __ldcg(p + m);
}
// the D1 values of one cell from global memory, streaming (evict-first) loads; 16-byte vectors
// when D1·sizeof(S) is a multiple of 16 (cells start at multiples of D1 values)
template <typename S, int D1>
__device__ __forceinline__ void load_cell_cs(const S* p, S* out, uint64_t pol) {
  if constexpr (sizeof(S) == 8 && D1 == 4) {  // one 32-byte load (sm_100 256-bit LDG), L1 bypass, L2 evict-first
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
        : "=d"(out[0]), "=d"(out[1]), "=d"(out[2]), "=d"(out[3])
        : "l"(p), "l"(pol));
  } else if constexpr ((D1 * sizeof(S)) % 16 == 0) {
    constexpr int NV = D1 * (int)sizeof(S) / 16;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if constexpr (sizeof(S) == 8) {
        const double2 x = __ldcs(reinterpret_cast<const double2*>(p) + v);
        out[2 * v] = x.x;
        out[2 * v + 1] = x.y;
      } else {
        const float4 x = __ldcs(reinterpret_cast<const float4*>(p) + v);
        out[4 * v] = x.x;
        out[4 * v + 1] = x.y;
        out[4 * v + 2] = x.z;
        out[4 * v + 3] = x.w;
      }
    }
  } else {
#pragma unroll
    for (int m = 0; m < D1; ++m) out[m] = __ldcs(p + m);
  }
}
// NC consecutive values at p (16-byte vectors when NC·sizeof(S) is a multiple of 16 and p is aligned)
template <typename S, int NC>
__device__ __forceinline__ void load_run(const S* p, S* out) {
  if constexpr ((NC * sizeof(S)) % 16 == 0) {
    constexpr int PER = 16 / (int)sizeof(S);
#pragma unroll
    for (int v = 0; v < NC / PER; ++v) {
      if constexpr (sizeof(S) == 8) {
        const double2 x = reinterpret_cast<const double2*>(p)[v];
        out[v * 2] = x.x;
        out[v * 2 + 1] = x.y;
      } else {
        const float4 x = reinterpret_cast<const float4*>(p)[v];
        out[v * 4] = x.x;
        out[v * 4 + 1] = x.y;
        out[v * 4 + 2] = x.z;
        out[v * 4 + 3] = x.w;
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < NC; ++c) out[c] = p[c];
  }
}

struct Meta {
  uint32_t e0, e1, f0, f1;
};
template <typename S>
__device__ __forceinline__ Meta meta(const CellArgs<S>& A, int64_t row, int64_t lim) {
  Meta m{0u, 0u, 0u, 0u};
  if (row < lim) {
    m.e0 = (uint32_t)__ldg(A.row_nz + row);
    m.e1 = (uint32_t)__ldg(A.row_nz + row + 1);
    m.f0 = (uint32_t)__ldg(A.row_fib + row);
    m.f1 = (uint32_t)__ldg(A.row_fib + row + 1);
  }
  return m;
}

// u at a nonzero's column: from a per-group shared copy of the row's fiber u (one shared load
// per nonzero).  Round 1 measured shuffles from the fiber lanes faster for fp64 Newton with
// FREG = 2 (0.84 vs 0.92 ms); with the packed Newton record (one gather per cell) the shared
// copy wins there too (cfg4 fused 0.675 -> 0.649 ms), so every instance uses it.
template <typename S, int FREG, int JAC>
__host__ __device__ constexpr bool cells_su() {
  return true;
}

// C32: the D_u w rows are 32-byte aligned and read with one 256-bit load each (a compile-time
// choice: a runtime branch between load widths makes the merged result wait on the load at once)
// COH: the chain records are read through L2 only (ld.global.cg), not the non-coherent
// read-only path — the single-pass step kernel writes them during the same launch.
// Rows row, row + NG, ... < lim of one group; wrow0 is the first row of the group's warp.
// PM: the row's per-cell data comes from the packed 64-bit words (ck_m / ck_kb), loaded one row
// ahead straight into registers — no shared-memory staging of K and (fiber, position) slices.
template <typename S, int D1, int G, int CPL, int FREG, bool DO_R, int JAC, bool WB, bool C32, bool COH,
          bool PM = false>
__device__ __forceinline__ void cell_rows(const CellArgs<S>& A, int64_t row, const int64_t wrow0, const int64_t NG,
                                          const int64_t lim) {
  constexpr bool kN = JAC == kJacNewtonP0 || JAC == kJacNewtonPK;
  constexpr bool kPK = JAC == kJacNewtonPK;
  constexpr bool SU = cells_su<S, FREG, JAC>() && (DO_R || kN);
  static_assert(!(PM && WB), "packed row words replace the staged slices");
  using L = CellSmem<S, D1, G, CPL, JAC != kJacNone, SU ? G * FREG : 0, PM>;
  constexpr bool kJ = JAC != kJacNone;
  constexpr bool kU = DO_R || kN;  // u (and B_iK) needed; the Picard matrix alone reads no u
  // Control flow is warp-uniform (a group past the last row runs on an empty one), so
  // every shuffle uses the full mask with width G.
  constexpr unsigned FM = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x % G;
  const int grp = threadIdx.x / G;
  // WB: the warp's region holds its two stages, its groups' s_t and its mbarriers
  unsigned char* gs = WB ? smem + (threadIdx.x >> 5) * L::wbytes : smem + grp * L::bytes;
  const uint32_t gs_s = smem_u32(gs);
  S* s_t = reinterpret_cast<S*>(WB ? gs + L::wo_t + (grp % L::WPG) * L::CE * (int)sizeof(S) : gs + L::o_t);
  uint64_t* bars = reinterpret_cast<uint64_t*>(gs + L::wo_bar);
  S* s_u = reinterpret_cast<S*>(WB ? gs + L::wo_u + (grp % L::WPG) * G * FREG * (int)sizeof(S) : gs + L::o_u);
  constexpr int STG = WB ? L::wstage : L::stage;
  constexpr int SK = WB ? L::w_k : L::st_k, SV = WB ? L::w_v : L::st_v, SB = WB ? L::w_b : L::st_b;
  const uint64_t pol = evict_first_policy();

  // fiber lanes: lane f holds fiber f (+ G, + 2G, ...): its column and canonical start (loaded
  // two rows ahead) and u at its column (one row ahead), so no load waits on another in-row
  auto fibers = [&](const Meta& m, int* fj, int* fb) {
#pragma unroll
    for (int q = 0; q < FREG; ++q) {
      const int f = lane + q * G;
      const bool ok = f < (int)(m.f1 - m.f0);
      fj[q] = ((kU || kJ) && ok) ? __ldg(A.fib_j + m.f0 + f) : -1;
      fb[q] = ok ? (int)__ldg(A.fib_nz + m.f0 + f) : 0;  // raw offset: e0 is subtracted at use (no stall now)
    }
  };
  // unconditional (clamped) loads: a select on the loaded value would stall right here; the
  // value of a lane without a fiber is never shuffled out
  auto ucols = [&](const int* fj, S* uj) {
#pragma unroll
    for (int q = 0; q < FREG; ++q) uj[q] = kU ? __ldg(A.u + (fj[q] >= 0 ? fj[q] : 0)) : S(0);
  };
  // stage buffer b <- this group's row slices.  cp.async: every lane copies 16-byte chunks of
  // its group's row.  WB: the warp's rows are consecutive, so lane 0 of the warp copies the
  // warp's contiguous spans with three TMA bulk copies completing on bars[b]; each group then
  // addresses its row at its offset inside the span.
  auto stage_in = [&](int b, const Meta& m, int& sk, int& sv, int& sb) {
    const uint32_t dst = gs_s + b * STG;
    if constexpr (WB) {
      const uint32_t e0w = __shfl_sync(FM, m.e0, 0);
      const uint32_t e1w = __reduce_max_sync(FM, m.e1);  // rows past the end have e1 = 0
      const int n = (int)(e1w - e0w);
      const char *lk, *lv, *lb;
      uint32_t nk, nv, nb;
      const int o = (int)(m.e0 - e0w);  // this group's row inside the warp span (ne = 0 past the end)
      sk = span16(A.ck_k + e0w / D1, n / D1, &lk, &nk) + o / D1;
      sv = span16(A.ck_val + e0w, n, &lv, &nv) + o;
      sb = span16(A.ck_b + e0w, n, &lb, &nb) + o;
      if ((threadIdx.x & 31) == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of the buffer
        bar_expect(&bars[b], nk + nv + nb);
        if (nk) bulk_copy(dst + SK, lk, nk, &bars[b], pol);
        if (nv) bulk_copy(dst + SV, lv, nv, &bars[b], pol);
        if (nb) bulk_copy(dst + SB, lb, nb, &bars[b], pol);
      }
    } else {
      const int n = (int)(m.e1 - m.e0);
      sk = stage_span<uint32_t, G, L::CC>(dst + SK, A.ck_k + m.e0 / D1, n / D1, lane, pol);
      sv = 0;  // values: read straight into registers (below)
      sb = stage_span<uint16_t, G, L::CE>(dst + SB, A.ck_b + m.e0, n, lane, pol);
      commit();
    }
  };
  // PM: the lane's packed words of a row (streamed once: L1 bypass, L2 evict-first) and the row's
  // first K; a lane past the row's cells holds 0 and never uses it
  auto words = [&](const Meta& m, int64_t r, uint64_t* mw, uint32_t& kb) {
    const int n = (int)(m.e1 - m.e0) / D1;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int q = lane + c * G;
      uint64_t x = 0;
      if (q < n)
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
            : "=l"(x)
            : "l"(A.ck_m + m.e0 / D1 + q), "l"(pol));
      mw[c] = x;
    }
    kb = r < lim ? __ldg(A.ck_kb + r) : 0u;
  };
  if constexpr (WB) {
    if ((threadIdx.x & 31) == 0) {
      bar_init(&bars[0]);
      bar_init(&bars[1]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  uint32_t phase = 0;  // WB: parity bit per buffer

  Meta cur = meta(A, row, lim);
  Meta nxt = meta(A, row + NG, lim);
  Meta nn = meta(A, row + 2 * NG, lim);
  int shk = 0, shv = 0, shb = 0;
  uint64_t mw_cur[PM ? CPL : 1], mw_nxt[PM ? CPL : 1];
  uint32_t kb_cur = 0, kb_nxt = 0;
  if constexpr (PM) words(cur, row, mw_cur, kb_cur);
  else stage_in(0, cur, shk, shv, shb);
  S uj_cur[FREG], uj_nxt[FREG];
  int fb_cur[FREG], fb_nxt[FREG], fj_cur[FREG], fj_nxt[FREG];
  fibers(cur, fj_cur, fb_cur);
  fibers(nxt, fj_nxt, fb_nxt);
  ucols(fj_cur, uj_cur);
  int st = 0;
  for (int64_t wr = wrow0; wr < lim; wr += NG, row += NG) {
    const int ne = (int)(cur.e1 - cur.e0);
    const int nc = ne / D1;
    const int nf = (int)(cur.f1 - cur.f0);
    // ---- prefetch: the next row's stream (async) and fiber data, metadata two rows ahead
    int nshk = 0, nshv = 0, nshb = 0;
    if constexpr (PM) words(nxt, row + NG, mw_nxt, kb_nxt);
    else if (WB || row + NG < lim) stage_in(st ^ 1, nxt, nshk, nshv, nshb);  // WB: 0-byte arrive past the end
    else commit();
    ucols(fj_nxt, uj_nxt);
    int fj_nn[FREG], fb_nn[FREG];
    fibers(nn, fj_nn, fb_nn);
    const Meta n3 = meta(A, row + 3 * NG, lim);
    if constexpr (!WB && JAC == kJacNone) {
      // apply-only: the values of a row go straight to registers when its turn comes; one bulk L2
      // prefetch per warp of its rows' contiguous value span two steps ahead, so that load waits
      // on L2, not HBM (cfg4 fp64 apply 0.411 -> 0.373 ms).  The Jacobian kernels are LSU-bound,
      // not waiting on HBM: the same prefetch measured slower there (fused 0.715 -> 0.72-0.795 ms).
      if (A.pf) {
        const uint32_t pe0 = __shfl_sync(FM, nn.e0, 0);
        const uint32_t pe1 = __reduce_max_sync(FM, nn.e1);
        if ((threadIdx.x & 31) == 0 && pe1 > pe0) {
          const char* lo;
          uint32_t nb;
          span16(A.ck_val + pe0, (int)(pe1 - pe0), &lo, &nb);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(nb) : "memory");
        }
      }
    }
    if constexpr (WB) {
      bar_wait(&bars[st], (phase >> st) & 1u);
      phase ^= 1u << st;
    } else if constexpr (!PM) {
      wait_prev();
    }
    __syncwarp();
    const unsigned char* cs = gs + st * STG;
    const uint32_t* bk = reinterpret_cast<const uint32_t*>(cs + SK) + shk;
    const S* bv = reinterpret_cast<const S*>(cs + SV) + shv;
    const uint16_t* bb = reinterpret_cast<const uint16_t*>(cs + SB) + shb;
    // ---- the lane's cell values (cp.async path: streamed straight into registers, issued with
    // the gathers below so their latencies overlap; a lane past the row's cells reads cell 0)
    S tvg[WB ? 1 : CPL][D1];
    if constexpr (!WB) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int q = lane + c * G;
        const S* pv = A.ck_val + (q < nc ? (size_t)cur.e0 + (size_t)q * D1 : (size_t)0);
        load_cell_cs<S, D1>(pv, tvg[c], pol);
      }
    }
    // ---- gathers of the lane's cells: w_K and (D_u w)_{K, 0..d}, all in flight together
    S wk[CPL];
    S dd[kN ? CPL : 1][D1];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int q = lane + c * G;
      const bool ok = q < nc;
      uint32_t K;
      if constexpr (PM) K = ok ? kb_cur + (uint32_t)(mw_cur[c] >> A.ks) : 0u;
      else K = ok ? bk[q] : 0u;
      // PM: no select on a loaded value here (in the PM instances it stalled the warp at once:
      // fused 0.70 -> 0.64 ms on cfg4); a lane past the row's cells loads a valid cell's data and
      // every use below is predicated on ok.  The staged instances keep the select (measured
      // faster there: 0.67 vs 0.70 ms) — the two forms give the same sums.
      if constexpr (!kPK) wk[c] = PM ? __ldg(A.w + K) : ok ? __ldg(A.w + K) : S(0);
      if constexpr (kN) {
        // the cell's D1 values (16-byte vector loads); a lane past the row's cells loads cell 0's
        // row and never uses it (no select on the loaded value)
        if constexpr (COH) {
          load_cell_cg<S, D1>(A.chain + (size_t)K * D1, dd[c], C32);
        } else if constexpr ((D1 * sizeof(S)) % 16 == 0) {
          load_cell_ldg<S, D1>(A.chain + (size_t)K * D1, dd[c], C32);
        } else {
#pragma unroll
          for (int m = 0; m < D1; ++m) dd[c][m] = __ldg(A.chain + (size_t)K * D1 + m);
        }
        if constexpr (kPK) {  // packed record [w_K, D_0 .. D_{d−1}]: D_d = −Σ_{m<d} D_m
          wk[c] = PM ? dd[c][0] : ok ? dd[c][0] : S(0);
          S sd = S(0);
#pragma unroll
          for (int m = 0; m + 1 < D1; ++m) {
            dd[c][m] = dd[c][m + 1];
            sd = xadd(sd, dd[c][m]);
          }
          dd[c][D1 - 1] = -sd;
        }
      }
    }
    const bool vec_v = (reinterpret_cast<uintptr_t>(bv) & 15u) == 0;
    if constexpr (SU && kU) {  // u at the row's fibers, for one shared load per nonzero
#pragma unroll
      for (int q = 0; q < FREG; ++q) s_u[lane + q * G] = uj_cur[q];
      __syncwarp();
    }
    // the diagonal fiber (i, i): one nonzero per cell of the row — summed in registers
    int fd = -1;
    if constexpr (kJ) {
      const int64_t irow = row + A.diag_off;
      const int goff = (threadIdx.x & 31) & ~(G - 1);
      constexpr unsigned GM = (G == 32) ? 0xffffffffu : ((1u << G) - 1u);
#pragma unroll
      for (int q = 0; q < FREG; ++q) {
        const unsigned b = (__ballot_sync(FM, lane + q * G < nf && fj_cur[q] == irow) >> goff) & GM;
        if (b) fd = q * G + __ffs(b) - 1;
      }
    }
    S dacc = S(0);
    S acc = S(0);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int q = lane + c * G;
      const bool ok = q < nc;
      S tv[D1];
      uint32_t bq[D1];
      if (ok) {
        if constexpr (WB) {
          load_cell<S, D1>(bv + q * D1, vec_v, tv);
        } else {
#pragma unroll
          for (int m = 0; m < D1; ++m) tv[m] = tvg[c][m];
        }
        if constexpr (PM) {  // (fiber, position) fields of the packed word, re-packed as in ck_b
          const uint32_t fmk = (1u << A.fb) - 1u, pmk = (1u << (A.fw - A.fb)) - 1u;
#pragma unroll
          for (int m = 0; m < D1; ++m) {
            const uint32_t x = (uint32_t)(mw_cur[c] >> (m * A.fw));
            bq[m] = (x & fmk) | (((x >> A.fb) & pmk) << kCkPosShift);
          }
        } else if constexpr (D1 == 4) {
          const uint2 x = *reinterpret_cast<const uint2*>(bb + q * D1);  // 8-byte aligned: e0 % 4 == 0
          bq[0] = x.x & 0xffffu;
          bq[1] = x.x >> 16;
          bq[2] = x.y & 0xffffu;
          bq[3] = x.y >> 16;
        } else {
#pragma unroll
          for (int m = 0; m < D1; ++m) bq[m] = bb[q * D1 + m];
        }
      } else {
#pragma unroll
        for (int m = 0; m < D1; ++m) {
          tv[m] = S(0);
          bq[m] = 0u;
        }
      }
      S B = S(0);
      if constexpr (kU) {
#pragma unroll
        for (int m = 0; m < D1; ++m) {
          const int fid = (int)(bq[m] & kCkFibMask);
          S um;
          if constexpr (SU) {
            um = s_u[fid];
          } else {
            um = __shfl_sync(FM, uj_cur[0], fid % G, G);
#pragma unroll
            for (int x = 1; x < FREG; ++x) {
              const S y = __shfl_sync(FM, uj_cur[x], fid % G, G);
              um = (fid / G == x) ? y : um;
            }
          }
          B = (m == 0) ? xmul(tv[m], um) : xfma(tv[m], um, B);
        }
      }
      if constexpr (DO_R) {
        if (!PM || ok) acc = xfma(wk[c], B, acc);
      }
      if constexpr (kJ) {
        if (ok) {
#pragma unroll
          for (int m = 0; m < D1; ++m) {
            S t = xmul(tv[m], wk[c]);
            if constexpr (kN) t = xfma(B, dd[c][m], t);
            if ((int)(bq[m] & kCkFibMask) == fd) dacc = xadd(dacc, t);
            else s_t[bq[m] >> kCkPosShift] = t;
          }
        }
      }
    }
    if constexpr (DO_R) {
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) acc = xadd(acc, __shfl_xor_sync(FM, acc, o, G));
      if (lane == 0 && row < lim) A.r[row] = acc;
    }
    if constexpr (kJ) {
      // ---- diagonal: lane partials (cell order) + butterfly; the other fibers: their lane sums
      // the scattered terms in canonical order (a handful per fiber: the cells around an edge)
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) dacc = xadd(dacc, __shfl_xor_sync(FM, dacc, o, G));
      if (lane == 0 && fd >= 0) A.csr[cur.f0 + fd] = dacc;
      __syncwarp();  // the scatter into s_t is complete
#pragma unroll
      for (int q = 0; q < FREG; ++q) {
        const int f = lane + q * G;
        const int fs = fb_cur[q] - (int)cur.e0;
        const int nx_same = __shfl_sync(FM, fs, (lane + 1) % G, G);
        const int nx_next = (q + 1 < FREG) ? __shfl_sync(FM, fb_cur[(q + 1) % FREG] - (int)cur.e0, 0, G) : ne;
        if (f < nf && f != fd) {
          const int yb = (f + 1 >= nf) ? ne : (lane + 1 < G ? nx_same : nx_next);
          // the first 8 terms loaded together (independent shared loads), summed in order; a
          // longer fiber (unstructured meshes) continues serially
          S v[8];
#pragma unroll
          for (int x = 0; x < 8; ++x) v[x] = (fs + x < yb) ? s_t[fs + x] : S(0);
          S a = S(0);
#pragma unroll
          for (int x = 0; x < 8; ++x)
            if (fs + x < yb) a = xadd(a, v[x]);
          for (int y = fs + 8; y < yb; ++y) a = xadd(a, s_t[y]);
          A.csr[cur.f0 + f] = a;
        }
      }
    }
    __syncwarp();  // stage st and s_t are free for reuse
    cur = nxt;
    nxt = nn;
    nn = n3;
    if constexpr (PM) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) mw_cur[c] = mw_nxt[c];
      kb_cur = kb_nxt;
    }
    shk = nshk;
    shv = nshv;
    shb = nshb;
#pragma unroll
    for (int q = 0; q < FREG; ++q) {
      uj_cur[q] = uj_nxt[q];
      fb_cur[q] = fb_nxt[q];
      fb_nxt[q] = fb_nn[q];
      fj_cur[q] = fj_nxt[q];
      fj_nxt[q] = fj_nn[q];
    }
    st ^= 1;
  }
}

template <typename S, int D1, int G, int CPL, int FREG, bool DO_R, int JAC, bool WB, bool C32 = false, bool PM = false>
__global__ void __launch_bounds__(cell_threads<S, JAC>(),
                                  (JAC == kJacNone || G >= 16) ? 3 * 256 / cell_threads<S, JAC>() : 2 * 256 / cell_threads<S, JAC>())
    k_cell(const CellArgs<S> A) {
  constexpr int GPB = cell_threads<S, JAC>() / G;
  const int64_t NG = (int64_t)gridDim.x * GPB;
  const int64_t row = (int64_t)blockIdx.x * GPB + threadIdx.x / G;
  const int64_t wrow0 = (int64_t)blockIdx.x * GPB + (threadIdx.x >> 5) * (32 / G);
  if (wrow0 >= A.n_u) return;
  cell_rows<S, D1, G, CPL, FREG, DO_R, JAC, WB, C32, false, PM>(A, row, wrow0, NG, A.n_u);
}

// Offline: the cell-major copy of a P0-W tensor's rows (one thread per row).
template <typename S>
__global__ void k_make_cells(int64_t n_u, const int64_t* __restrict__ row_fib, const uint32_t* __restrict__ fib_nz,
                             const uint32_t* __restrict__ nz_k, const uint8_t* __restrict__ nz_aux,
                             const S* __restrict__ nz_val, int D1, uint32_t* ck_k, S* ck_val, uint16_t* ck_b, int* err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_u) return;
  const int64_t f0 = row_fib[i], f1 = row_fib[i + 1];
  const uint32_t e0 = fib_nz[f0], e1 = fib_nz[f1];
  if ((e1 - e0) % D1 != 0 || e0 % D1 != 0 || e1 - e0 > (uint32_t)kCellsMaxNnz || f1 - f0 > kCkFibMask + 1) {
    atomicExch(err, 1);
    return;
  }
  for (int64_t f = f0; f < f1; ++f)
    for (uint32_t e = fib_nz[f]; e < fib_nz[f + 1]; ++e) {
      const uint32_t slot = nz_aux[e];
      const uint32_t loc = (nz_k[e] >> kKShift) & 3u;
      const uint32_t idx = e0 + slot * D1 + loc;
      if (loc >= (uint32_t)D1 || idx >= e1) {
        atomicExch(err, 1);
        return;
      }
      ck_val[idx] = nz_val[e];
      ck_b[idx] = (uint16_t)((uint32_t)(f - f0) | ((e - e0) << kCkPosShift));
      if (loc == 0) ck_k[e0 / D1 + slot] = nz_k[e] & kKMask;
    }
}

// Offline: the packed row words (egfem_tensor::ck_m) from the cell-major copy, one thread per row.
// mode 0: the largest K − (row's first K) into *maxd; mode 1: write the words.
__global__ void k_make_words(int64_t n_u, const int64_t* __restrict__ row_nz, const uint32_t* __restrict__ ck_k,
                             const uint16_t* __restrict__ ck_b, int D1, int fb, int ks, int mode,
                             unsigned long long* maxd, uint64_t* ck_m, uint32_t* ck_kb) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_u) return;
  const int64_t c0 = row_nz[i] / D1, c1 = row_nz[i + 1] / D1;
  const uint32_t kb = c1 > c0 ? ck_k[c0] : 0u;
  if (mode == 0) {
    if (c1 > c0) atomicMax(maxd, (unsigned long long)(ck_k[c1 - 1] - kb));
    return;
  }
  ck_kb[i] = kb;
  const int fw = ks / D1;
  for (int64_t c = c0; c < c1; ++c) {
    uint64_t x = (uint64_t)(ck_k[c] - kb) << ks;
    for (int m = 0; m < D1; ++m) {
      const uint32_t b = ck_b[c * D1 + m];
      x |= (uint64_t)((b & kCkFibMask) | ((b >> kCkPosShift) << fb)) << (m * fw);
    }
    ck_m[c] = x;
  }
}

int g_sm_count[64] = {0};

// Row-stream staging: TMA bulk copies of each warp's consecutive rows (WB) when a warp holds
// at least 8 rows (G <= 4: the copies are large, measured faster on cfg3: fused 0.139 ->
// 0.107 ms), per-lane cp.async otherwise (cfg4, 4 rows per warp: 0.87 vs 0.94 ms with WB).
// EGFEM_CELLS_STAGE=cp|bulk forces one (experiments).
// Warp-level TMA staging pays off for narrow groups (many rows per warp) of fp32 rows; with fp64
// the per-lane path (values straight to registers, small shared footprint) measured faster
// (cfg3 fused 0.107 -> 0.103 ms), with fp32 the bulk path (apply 0.043 -> 0.038 ms).
bool cells_warp_bulk(int G, int vbytes) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EGFEM_CELLS_STAGE");
    v = (e && e[0] == 'b') ? 1 : (e && e[0] == 'c') ? 0 : 2;
  }
  return v == 2 ? (G <= 4 && vbytes == 4) : (v == 1);
}

// The packed 64-bit row words (PM kernels) when the tensor has them; EGFEM_CELLS_WORDS=0 keeps the
// staged (K, fiber|pos) slices (A/B experiments; both give bitwise the same results).
bool cells_packed_words() {
  static int v = -1;
  if (v < 0) v = getenv("EGFEM_CELLS_WORDS") ? (atoi(getenv("EGFEM_CELLS_WORDS")) != 0) : 1;
  return v;
}

template <typename S, int D1, int G, int CPL, int FREG, bool DO_R, int JAC>
egfem_status run_cells(const egfem_tensor* t, const CellArgs<S>& A, cudaStream_t s) {
  constexpr bool SU = cells_su<S, FREG, JAC>() && (DO_R || JAC == kJacNewtonP0 || JAC == kJacNewtonPK);
  using L = CellSmem<S, D1, G, CPL, JAC != kJacNone, SU ? G * FREG : 0>;
  using LP = CellSmem<S, D1, G, CPL, JAC != kJacNone, SU ? G * FREG : 0, true>;
  const bool wb = cells_warp_bulk(G, (int)sizeof(S));
  const bool pm = !wb && A.ck_m && cells_packed_words();
  auto fn = wb ? k_cell<S, D1, G, CPL, FREG, DO_R, JAC, true>
               : pm ? k_cell<S, D1, G, CPL, FREG, DO_R, JAC, false, false, true> : k_cell<S, D1, G, CPL, FREG, DO_R, JAC, false>;
  if constexpr ((JAC == kJacNewtonP0 || JAC == kJacNewtonPK) && D1 == 4 && sizeof(S) == 8) {
    if (A.chain32)
      fn = wb ? k_cell<S, D1, G, CPL, FREG, DO_R, JAC, true, true>
              : pm ? k_cell<S, D1, G, CPL, FREG, DO_R, JAC, false, true, true> : k_cell<S, D1, G, CPL, FREG, DO_R, JAC, false, true>;
  }
  constexpr int CT = cell_threads<S, JAC>();
  const int smem = wb ? L::wbytes * (CT / 32) : pm ? LP::bytes * (CT / G) : L::bytes * (CT / G);
  if (smem > 48 * 1024) EGFEM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  static int carve = -2;  // EGFEM_CELLS_CARVE=<percent>: preferred shared-memory carveout (experiments)
  if (carve == -2) carve = getenv("EGFEM_CELLS_CARVE") ? atoi(getenv("EGFEM_CELLS_CARVE")) : -1;
  if (carve >= 0) EGFEM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
  const int dev = t->device & 63;
  if (!g_sm_count[dev])
    EGFEM_CUDA_TRY(cudaDeviceGetAttribute(&g_sm_count[dev], cudaDevAttrMultiProcessorCount, t->device));
  int per_sm = 0;
  EGFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, CT, smem));
  const int64_t need = (t->n_u + (CT / G) - 1) / (CT / G);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)std::max(per_sm, 1) * g_sm_count[dev]));
  fn<<<grid, CT, smem, s>>>(A);
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

template <typename S, int D1, int G, int CPL, int FREG>
egfem_status cells_mode(const egfem_tensor* t, const CellArgs<S>& A, bool do_r, int jac, bool packed,
                        cudaStream_t s) {
  if (do_r) {
    if (jac == kJacNone) return run_cells<S, D1, G, CPL, FREG, true, kJacNone>(t, A, s);
    if (jac == kJacPicard) return run_cells<S, D1, G, CPL, FREG, true, kJacPicard>(t, A, s);
    if (packed) return run_cells<S, D1, G, CPL, FREG, true, kJacNewtonPK>(t, A, s);
    return run_cells<S, D1, G, CPL, FREG, true, kJacNewtonP0>(t, A, s);
  }
  if (jac == kJacPicard) return run_cells<S, D1, G, CPL, FREG, false, kJacPicard>(t, A, s);
  if (packed) return run_cells<S, D1, G, CPL, FREG, false, kJacNewtonPK>(t, A, s);
  return run_cells<S, D1, G, CPL, FREG, false, kJacNewtonP0>(t, A, s);
}

// (G, CPL, FREG) per dimension: the first configuration that holds the longest row's
// cells and fibers.  EGFEM_CELLS_CFG="G,CPL" picks another listed one (experiments).
struct CellCfg {
  int d1, G, CPL, FREG;
};
constexpr CellCfg kCellCfgs[] = {{3, 2, 3, 4}, {3, 4, 4, 8}, {3, 16, 3, 1}, {4, 8, 3, 2},
                                 {4, 16, 3, 2}, {4, 16, 4, 4}, {4, 32, 3, 1}};

bool pick_cells(const egfem_tensor* t, CellCfg* out) {
  static int envG = -1, envC = -1;
  if (envG < 0) {
    envG = envC = 0;
    if (const char* e = getenv("EGFEM_CELLS_CFG")) sscanf(e, "%d,%d", &envG, &envC);
  }
  const int d1 = t->dim + 1;
  const int mc = t->max_row_nnz / d1;
  for (int pass = 0; pass < 2; ++pass)
    for (const CellCfg& c : kCellCfgs) {
      if (c.d1 != d1 || c.G * c.CPL < mc || c.G * c.FREG < t->max_row_fib) continue;
      if (pass == 0 && envG > 0 && (c.G != envG || c.CPL != envC)) continue;
      *out = c;
      return true;
    }
  return false;
}

template <typename S>
egfem_status cells_dispatch(const egfem_tensor* t, bool do_r, int jac, bool packed, const void* u, const void* w,
                            const void* chain, void* r, void* csr, cudaStream_t s) {
  CellArgs<S> A;
  A.n_u = t->n_u;
  A.row_nz = t->row_nz;
  A.row_fib = t->row_fib;
  A.fib_j = t->fib_j;
  A.fib_nz = t->fib_nz;
  A.ck_k = t->ck_k;
  A.ck_val = static_cast<const S*>(t->ck_val);
  A.ck_b = t->ck_b;
  A.ck_m = t->ck_m;
  A.ck_kb = t->ck_kb;
  A.fb = t->ck_fb;
  A.fw = t->ck_fb + t->ck_pb;
  A.ks = t->ck_ks;
  A.u = static_cast<const S*>(u);
  A.w = static_cast<const S*>(w);
  A.chain = static_cast<const S*>(chain);
  A.r = static_cast<S*>(r);
  A.csr = static_cast<S*>(csr);
  A.diag_off = t->row_begin - t->col_begin;
  A.chain32 = (reinterpret_cast<uintptr_t>(chain) & 31u) == 0;
  static int pf_env = -1;
  if (pf_env < 0) pf_env = getenv("EGFEM_CELLS_PF") ? (atoi(getenv("EGFEM_CELLS_PF")) != 0) : 1;
  A.pf = pf_env;
  CellCfg c{};
  if (!pick_cells(t, &c)) {
    set_error("no cell-major configuration");
    return EGFEM_ERR_UNSUPPORTED;
  }
  if (getenv("EGFEM_DEBUG"))
    fprintf(stderr, "[egfem] k_cell d1=%d G=%d CPL=%d FREG=%d do_r=%d jac=%d\n", c.d1, c.G, c.CPL, c.FREG, (int)do_r, jac);
#define EGFEM_CC(D_, G_, C_, F_) \
  if (c.d1 == D_ && c.G == G_ && c.CPL == C_) return cells_mode<S, D_, G_, C_, F_>(t, A, do_r, jac, packed, s);
  EGFEM_CC(3, 2, 3, 4)
  EGFEM_CC(3, 4, 4, 8)
  EGFEM_CC(3, 16, 3, 1)
  EGFEM_CC(4, 8, 3, 2)
  EGFEM_CC(4, 16, 3, 2)
  EGFEM_CC(4, 16, 4, 4)
  EGFEM_CC(4, 32, 3, 1)
#undef EGFEM_CC
  set_error("no cell-major configuration");
  return EGFEM_ERR_UNSUPPORTED;
}


// ------------------------------------------------------------------ single-pass Newton step
// step (1) of the gradient kinds and steps (2)+(3)
// (L183, L290–292) in ONE launch.  The work is a fixed sequence of items (StepPlan.seq): interp
// items (CI consecutive cells: w_K and the packed record [w_K, ∂w/∂u_0..∂w/∂u_{d−1}]) and row
// items (RI consecutive rows: r and the Newton Jacobian row values from the records of the
// rows' cells).  Warps take items in sequence order from a global counter.  A row item is placed
// after every interp item that produces a record it reads (+ a lag), waits on those items'
// release flags and reads the records through L2 (COH loads).  Deadlock-free for any residency:
// an item waits only on items earlier in the sequence, which were taken by warps that are
// already running and never wait on later items.  The records a row item reads were written
// moments earlier (one mesh layer ahead), so they are gathered from L2, and the interp's
// gathers and FP64 work overlap the row items' streaming in the same SMs.  The flags carry the
// launch's epoch (no reset between launches, so the step is CUDA-graph capturable); the last
// warp to finish rewinds the counters and advances the epoch.
template <typename S>
struct StepArgs {
  const double* coords;
  const float* coordsf;
  const int32_t* cells;
  int64_t n_cells;
  S* w;
  S* chain;
  double p;
  bool minsurf;
  const int32_t* seq;   // item order: >= 0 interp item, < 0 row item ~r
  const int32_t* need;  // per row item: first and last interp item it reads
  uint32_t* sync;       // [0] item counter, [1] finished warps, [2] epoch, [4..] interp item flags
  int n_items;
  int CI, RI;
  bool nowait;          // diagnostics (EGFEM_STEP_MODE=2: row items only, no waiting)
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename S, int D1, int G, int CPL, int FREG, bool C32, bool CF, bool PM = false>
__global__ void __launch_bounds__(cell_threads<S, kJacNewtonPK>(), 2 * 256 / cell_threads<S, kJacNewtonPK>())
    k_step(const CellArgs<S> A, const StepArgs<S> B) {
  constexpr int D = D1 - 1;
  constexpr int WPG = 32 / G;
  constexpr unsigned FM = 0xffffffffu;
  const int wl = threadIdx.x & 31;
  uint32_t* const flags = B.sync + 4;
  const uint32_t ep = *reinterpret_cast<volatile uint32_t*>(B.sync + 2) + 1u;
  for (;;) {
    uint32_t it = 0;
    if (wl == 0) it = atomicAdd(B.sync, 1u);
    it = __shfl_sync(FM, it, 0);
    if (it >= (uint32_t)B.n_items) break;
    const int code = __ldg(B.seq + it);
    if (code >= 0) {
      const int64_t c0 = (int64_t)code * B.CI;
      const int64_t c1 = min(c0 + (int64_t)B.CI, B.n_cells);
      ip::interp_cells<S, D, true, true, CF>(B.coords, B.coordsf, B.cells, B.cells, nullptr, c0 + wl, c1, 32, A.u,
                                               B.w, B.chain, B.p, B.minsurf, 1);
      __syncwarp();  // every lane's records are written (the release below is cumulative over them)
      if (wl == 0) st_release(flags + code, ep);
    } else {
      const int r = ~code;
      const int lo = __ldg(B.need + 2 * r), hi = __ldg(B.need + 2 * r + 1);
      if (!B.nowait)
        for (int q = lo + wl; q <= hi; q += 32)
          while (ld_acquire(flags + q) != ep) __nanosleep(64);
      __syncwarp();
      const int64_t base = (int64_t)r * B.RI;
      const int64_t lim = min(base + (int64_t)B.RI, A.n_u);
      cell_rows<S, D1, G, CPL, FREG, true, kJacNewtonPK, false, C32, true, PM>(A, base + wl / G, base, WPG, lim);
    }
  }
  __syncwarp();
  if (wl == 0) {
    const uint32_t total = gridDim.x * (blockDim.x / 32);
    __threadfence();
    if (atomicAdd(B.sync + 1, 1u) == total - 1u) {  // every other warp has left the item loop
      B.sync[0] = 0u;
      B.sync[1] = 0u;
      __threadfence();
      atomicAdd(B.sync + 2, 1u);
    }
  }
}

// per row item: the first and last interp item whose records its rows read
__global__ void k_step_need(int64_t n_u, const int64_t* __restrict__ row_nz, const uint32_t* __restrict__ ck_k, int d1,
                            int RI, int CI, int n_ritems, int32_t* need) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_ritems) return;
  uint32_t lo = 0xffffffffu, hi = 0u;
  bool any = false;
  for (int64_t i = (int64_t)r * RI; i < min((int64_t)(r + 1) * RI, n_u); ++i) {
    const int64_t a = row_nz[i] / d1, b = row_nz[i + 1] / d1;
    if (b <= a) continue;
    any = true;
    lo = min(lo, ck_k[a]);       // a row's cells are in ascending K
    hi = max(hi, ck_k[b - 1]);
  }
  need[2 * r] = any ? (int32_t)(lo / (uint32_t)CI) : 0;
  need[2 * r + 1] = any ? (int32_t)(hi / (uint32_t)CI) : -1;
}

template <typename S, int D1, int G, int CPL, int FREG, bool C32>
egfem_status run_step(const egfem_tensor* t, const CellArgs<S>& A, const StepArgs<S>& B, cudaStream_t s) {
  using L = CellSmem<S, D1, G, CPL, true, G * FREG>;
  using LP = CellSmem<S, D1, G, CPL, true, G * FREG, true>;
  const bool pm = A.ck_m && cells_packed_words();  // the row items read the packed row words too
  auto fn = B.coordsf ? (pm ? k_step<S, D1, G, CPL, FREG, C32, true, true> : k_step<S, D1, G, CPL, FREG, C32, true>)
                      : (pm ? k_step<S, D1, G, CPL, FREG, C32, false, true> : k_step<S, D1, G, CPL, FREG, C32, false>);
  constexpr int CT = cell_threads<S, kJacNewtonPK>();
  const int smem = (pm ? LP::bytes : L::bytes) * (CT / G);
  if (smem > 48 * 1024) EGFEM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int dev = t->device & 63;
  if (!g_sm_count[dev])
    EGFEM_CUDA_TRY(cudaDeviceGetAttribute(&g_sm_count[dev], cudaDevAttrMultiProcessorCount, t->device));
  int per_sm = 0;
  EGFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, CT, smem));
  const int grid = std::max(per_sm, 1) * g_sm_count[dev];
  fn<<<grid, CT, smem, s>>>(A, B);
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

}  // namespace

bool cells_path_ok(const egfem_tensor* t, int jac) {
  if (!t->ck_val || jac == 2 /* W = V Newton */) return false;
  CellCfg c{};
  return pick_cells(t, &c);
}

// how k_cell reads a row's per-cell data for this tensor (the variant run_cells picks)
const char* cells_variant(const egfem_tensor* t) {
  CellCfg c{};
  if (!pick_cells(t, &c)) return "no configuration";
  if (cells_warp_bulk(c.G, t->dtype == EGFEM_F64 ? 8 : 4)) return "warp TMA-staged slices";
  return (t->ck_m && cells_packed_words()) ? "packed 64-bit row words" : "cp.async-staged slices";
}

egfem_status launch_cells(const egfem_tensor* t, bool do_r, int jac, bool packed, const void* u, const void* w,
                          const void* chain, void* r, void* csr_vals, cudaStream_t s) {
  if (t->n_u <= 0) return EGFEM_OK;
  if (t->dtype == EGFEM_F64) return cells_dispatch<double>(t, do_r, jac, packed, u, w, chain, r, csr_vals, s);
  return cells_dispatch<float>(t, do_r, jac, packed, u, w, chain, r, csr_vals, s);
}

// Offline: cell-major copy for P0-W tensors of 2D/3D meshes whose rows fit the kernel;
// silently skipped otherwise (the canonical row / tile kernels then serve the tensor).
egfem_status make_p0_cells(egfem_tensor* t) {
  CellCfg cfg{};
  if (!t->has_mesh || !t->w_p0 || !t->nz_aux || (t->dim != 2 && t->dim != 3) || t->n_u <= 0 || t->nnz <= 0 ||
      t->max_row_nnz > kCellsMaxNnz || !pick_cells(t, &cfg))
    return EGFEM_OK;
  const int d1 = t->dim + 1;
  const size_t vs = t->dtype == EGFEM_F64 ? 8 : 4;
  EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->ck_k, 4 * (t->nnz / d1 + 1)));
  EGFEM_CUDA_TRY(dmalloc_padded(&t->ck_val, vs * t->nnz));
  EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->ck_b, 2 * t->nnz));
  int* err = nullptr;
  EGFEM_CUDA_TRY(cudaMalloc(&err, sizeof(int)));
  EGFEM_CUDA_TRY(cudaMemset(err, 0, sizeof(int)));
  const int nb = (int)((t->n_u + 127) / 128);
  if (t->dtype == EGFEM_F64)
    k_make_cells<double><<<nb, 128>>>(t->n_u, t->row_fib, t->fib_nz, t->nz_k, t->nz_aux, (const double*)t->nz_val, d1,
                                      t->ck_k, (double*)t->ck_val, t->ck_b, err);
  else
    k_make_cells<float><<<nb, 128>>>(t->n_u, t->row_fib, t->fib_nz, t->nz_k, t->nz_aux, (const float*)t->nz_val, d1,
                                     t->ck_k, (float*)t->ck_val, t->ck_b, err);
  count_launch();
  int herr = 0;
  cudaError_t ce = cudaMemcpy(&herr, err, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(err);
  EGFEM_CUDA_TRY(ce);
  if (getenv("EGFEM_DEBUG"))
    fprintf(stderr, "[egfem] cell-major copy: %s (n_u=%lld nnz=%lld max_row_nnz=%d max_row_fib=%d)\n",
            herr ? "rejected" : "built", (long long)t->n_u, (long long)t->nnz, t->max_row_nnz, t->max_row_fib);
  if (herr) {  // not cell-structured: drop the copy
    cudaFree(t->ck_k);
    cudaFree(t->ck_val);
    cudaFree(t->ck_b);
    t->ck_k = nullptr;
    t->ck_val = nullptr;
    t->ck_b = nullptr;
    return EGFEM_OK;
  }
  // packed row words: fiber and position fields as narrow as this tensor's rows allow, K as an
  // offset from the row's first cell in the remaining bits (skipped when it does not fit)
  auto bits = [](int n) {
    int b = 1;
    while ((1 << b) < n) ++b;
    return b;
  };
  const int fb = bits(t->max_row_fib), pb = bits(t->max_row_nnz), ks = d1 * (fb + pb);
  if (ks >= 64) return EGFEM_OK;
  unsigned long long* dmax = nullptr;
  EGFEM_CUDA_TRY(cudaMalloc(&dmax, sizeof(unsigned long long)));
  EGFEM_CUDA_TRY(cudaMemset(dmax, 0, sizeof(unsigned long long)));
  k_make_words<<<nb, 128>>>(t->n_u, t->row_nz, t->ck_k, t->ck_b, d1, fb, ks, 0, dmax, nullptr, nullptr);
  count_launch();
  unsigned long long hmax = 0;
  ce = cudaMemcpy(&hmax, dmax, sizeof(hmax), cudaMemcpyDeviceToHost);
  cudaFree(dmax);
  EGFEM_CUDA_TRY(ce);
  const bool fits = 64 - ks >= 32 || hmax < (1ull << (64 - ks));
  if (getenv("EGFEM_DEBUG"))
    fprintf(stderr, "[egfem] packed row words: fiber %d + position %d bits x %d, K offset max %llu in %d bits: %s\n", fb,
            pb, d1, hmax, 64 - ks, fits ? "built" : "skipped");
  if (!fits) return EGFEM_OK;
  EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->ck_m, 8 * (t->nnz / d1 + 1)));
  EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->ck_kb, 4 * (t->n_u + 1)));
  k_make_words<<<nb, 128>>>(t->n_u, t->row_nz, t->ck_k, t->ck_b, d1, fb, ks, 1, nullptr, t->ck_m, t->ck_kb);
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  t->ck_fb = fb;
  t->ck_pb = pb;
  t->ck_ks = ks;
  return EGFEM_OK;
}


struct StepPlan {
  int CI = 0, RI = 0, n_interp = 0, n_ritems = 0, n_items = 0, mode = 0;
  int32_t* seq = nullptr;
  int32_t* need = nullptr;
  uint32_t* sync = nullptr;
};

void free_step_plan(StepPlan* sp) {
  if (!sp) return;
  cudaFree(sp->seq);
  cudaFree(sp->need);
  cudaFree(sp->sync);
  delete sp;
}

// The item sequence of the single-pass step: interp items in cell order; row item r right after
// interp item need_hi(r) + lag (EGFEM_STEP_LAG, default 2048 items), so its records were
// produced a while before it is taken.  Opt-in: EGFEM_STEP=1 when the tensor is built (measured
// slower than the two launches on B200 — both halves are bound by the same load/store pipe,
// so egfem_step issues the two launches by default).  EGFEM_STEP_CI = cells per
// lane of an interp item (default 32: 1024 cells), EGFEM_STEP_RI = rows per row item (default 64).
egfem_status make_step_plan(egfem_tensor* t) {
  const char* en = getenv("EGFEM_STEP");
  if (!en || en[0] != '1') return EGFEM_OK;
  if (!t->ck_val || !t->has_mesh || !t->w_p0 || t->nwc != 1 || !t->wdofs_is_iota || !t->vdofs_is_cells ||
      (t->dim != 2 && t->dim != 3) || t->n_f != t->n_cells || t->row_begin != 0 ||
      t->col_begin != 0 || t->int_row_lo >= 0 || t->n_u <= 0 || t->n_cells <= 0)
    return EGFEM_OK;
  CellCfg c{};
  if (!pick_cells(t, &c)) return EGFEM_OK;
  const int m = getenv("EGFEM_STEP_CI") ? std::max(1, atoi(getenv("EGFEM_STEP_CI"))) : 32;
  int RI = getenv("EGFEM_STEP_RI") ? std::max(1, atoi(getenv("EGFEM_STEP_RI"))) : 64;
  RI = (RI + 15) / 16 * 16;  // a multiple of the groups per warp of every configuration
  const int lag = getenv("EGFEM_STEP_LAG") ? std::max(0, atoi(getenv("EGFEM_STEP_LAG"))) : 2048;
  const int64_t CI = 32LL * m;
  const int64_t n_interp = (t->n_cells + CI - 1) / CI, n_ritems = (t->n_u + RI - 1) / RI;
  if (n_interp + n_ritems >= (int64_t(1) << 31) - 1) return EGFEM_OK;
  StepPlan* sp = new StepPlan;
  sp->CI = (int)CI;
  sp->RI = RI;
  sp->n_interp = (int)n_interp;
  sp->n_ritems = (int)n_ritems;
  sp->n_items = (int)(n_interp + n_ritems);
  auto bail = [&](cudaError_t e) {
    free_step_plan(sp);
    set_error(std::string("step plan: ") + cudaGetErrorString(e));
    return EGFEM_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&sp->need, sizeof(int32_t) * 2 * n_ritems))) return bail(e);
  if ((e = cudaMalloc(&sp->seq, sizeof(int32_t) * sp->n_items))) return bail(e);
  if ((e = cudaMalloc(&sp->sync, sizeof(uint32_t) * (4 + n_interp)))) return bail(e);
  if ((e = cudaMemset(sp->sync, 0, sizeof(uint32_t) * (4 + n_interp)))) return bail(e);
  k_step_need<<<(int)((n_ritems + 127) / 128), 128>>>(t->n_u, t->row_nz, t->ck_k, t->dim + 1, RI, (int)CI,
                                                      (int)n_ritems, sp->need);
  count_launch();
  std::vector<int32_t> need(2 * n_ritems);
  if ((e = cudaMemcpy(need.data(), sp->need, sizeof(int32_t) * 2 * n_ritems, cudaMemcpyDeviceToHost))) return bail(e);
  // bucket the row items by the interp item they follow (-1: before every interp item)
  std::vector<int64_t> start(n_interp + 2, 0);
  auto key = [&](int64_t r) -> int64_t {
    const int64_t h = need[2 * r + 1];
    return h < 0 ? -1 : std::min<int64_t>(h + lag, n_interp - 1);
  };
  for (int64_t r = 0; r < n_ritems; ++r) ++start[key(r) + 2];
  for (int64_t q = 1; q < n_interp + 2; ++q) start[q] += start[q - 1];
  std::vector<int32_t> byk(n_ritems);
  {
    std::vector<int64_t> fill(start.begin(), start.end());
    for (int64_t r = 0; r < n_ritems; ++r) byk[fill[key(r) + 1]++] = (int32_t)r;
  }
  std::vector<int32_t> seq;
  seq.reserve(sp->n_items);
  for (int64_t x = start[0]; x < start[1]; ++x) seq.push_back(~byk[x]);
  for (int64_t q = 0; q < n_interp; ++q) {
    seq.push_back((int32_t)q);
    for (int64_t x = start[q + 1]; x < start[q + 2]; ++x) seq.push_back(~byk[x]);
  }
  if ((int64_t)seq.size() != sp->n_items) {  // cannot happen: every item is placed once
    free_step_plan(sp);
    return EGFEM_OK;
  }
  // diagnostics: EGFEM_STEP_MODE=1 runs the interp items only, =2 the row items only (no waits;
  // the records must exist from an earlier full step) — incomplete steps, for timing the parts
  sp->mode = getenv("EGFEM_STEP_MODE") ? atoi(getenv("EGFEM_STEP_MODE")) : 0;
  if (sp->mode == 1 || sp->mode == 2) {
    std::vector<int32_t> part;
    for (int32_t x : seq)
      if ((x >= 0) == (sp->mode == 1)) part.push_back(x);
    seq.swap(part);
    sp->n_items = (int)seq.size();
  }
  if ((e = cudaMemcpy(sp->seq, seq.data(), sizeof(int32_t) * seq.size(), cudaMemcpyHostToDevice))) return bail(e);
  if (getenv("EGFEM_DEBUG"))
    fprintf(stderr, "[egfem] step plan: %d interp items of %d cells, %d row items of %d rows, lag %d\n", sp->n_interp,
            sp->CI, sp->n_ritems, sp->RI, lag);
  t->step = sp;
  return EGFEM_OK;
}

bool step_path_ok(const egfem_tensor* t, egfem_interp_kind kind, const void* chain) {
  if (!t->step || !packed_chain_kind(kind)) return false;
  static const char* force = getenv("EGFEM_PATH");
  if (force && (force[0] == 't' || force[0] == 'r')) return false;
  // the 3D fp64 instances read each record with one 256-bit load: 32-byte aligned chain
  if (t->dim == 3 && t->dtype == EGFEM_F64 && (reinterpret_cast<uintptr_t>(chain) & 31u)) return false;
  CellCfg c{};
  return pick_cells(t, &c);
}

template <typename S>
egfem_status step_dispatch(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u, void* w,
                           void* chain, void* r, void* csr, cudaStream_t s) {
  CellArgs<S> A;
  A.n_u = t->n_u;
  A.row_nz = t->row_nz;
  A.row_fib = t->row_fib;
  A.fib_j = t->fib_j;
  A.fib_nz = t->fib_nz;
  A.ck_k = t->ck_k;
  A.ck_val = static_cast<const S*>(t->ck_val);
  A.ck_b = t->ck_b;
  A.ck_m = t->ck_m;
  A.ck_kb = t->ck_kb;
  A.fb = t->ck_fb;
  A.fw = t->ck_fb + t->ck_pb;
  A.ks = t->ck_ks;
  A.u = static_cast<const S*>(u);
  A.w = static_cast<const S*>(w);
  A.chain = static_cast<const S*>(chain);
  A.r = static_cast<S*>(r);
  A.csr = static_cast<S*>(csr);
  A.diag_off = 0;
  A.chain32 = (reinterpret_cast<uintptr_t>(chain) & 31u) == 0;
  A.pf = 0;
  StepArgs<S> B;
  B.coords = t->dim == 3 ? t->coords4 : t->coords;
  B.coordsf = t->coordsf;
  B.cells = t->cells;
  B.n_cells = t->n_cells;
  B.w = static_cast<S*>(w);
  B.chain = static_cast<S*>(chain);
  B.p = p;
  B.minsurf = kind == EGFEM_INTERP_MINSURF_P0;
  B.seq = t->step->seq;
  B.need = t->step->need;
  B.sync = t->step->sync;
  B.n_items = t->step->n_items;
  B.CI = t->step->CI;
  B.RI = t->step->RI;
  B.nowait = t->step->mode == 2;
  CellCfg c{};
  if (!pick_cells(t, &c)) return EGFEM_ERR_UNSUPPORTED;
  if (getenv("EGFEM_DEBUG"))
    fprintf(stderr, "[egfem] k_step d1=%d G=%d CPL=%d FREG=%d\n", c.d1, c.G, c.CPL, c.FREG);
#define EGFEM_SC(D_, G_, C_, F_)                                                     \
  if (c.d1 == D_ && c.G == G_ && c.CPL == C_) {                                      \
    if constexpr (D_ == 4 && sizeof(S) == 8) return run_step<S, D_, G_, C_, F_, true>(t, A, B, s); \
    else return run_step<S, D_, G_, C_, F_, false>(t, A, B, s);                      \
  }
  EGFEM_SC(3, 2, 3, 4)
  EGFEM_SC(3, 4, 4, 8)
  EGFEM_SC(3, 16, 3, 1)
  EGFEM_SC(4, 8, 3, 2)
  EGFEM_SC(4, 16, 3, 2)
  EGFEM_SC(4, 16, 4, 4)
  EGFEM_SC(4, 32, 3, 1)
#undef EGFEM_SC
  return EGFEM_ERR_UNSUPPORTED;
}

egfem_status launch_step(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u, void* w, void* chain,
                         void* r, void* csr_vals, cudaStream_t s) {
  if (!step_path_ok(t, kind, chain)) return EGFEM_ERR_UNSUPPORTED;
  if (t->dtype == EGFEM_F64) return step_dispatch<double>(t, kind, p, u, w, chain, r, csr_vals, s);
  return step_dispatch<float>(t, kind, p, u, w, chain, r, csr_vals, s);
}


}  // namespace egfem

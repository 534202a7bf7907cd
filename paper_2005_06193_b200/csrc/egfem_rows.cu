// Row-group kernel of libegfem.so (B200 / sm_100a): the fast path of steps (2)+(3).
//
// A group of G lanes (G = 8, 16 or 32, chosen from the longest row) walks rows
// grid-stride (the rows in flight stay one compact window, which keeps the w / D_u w
// gathers L2-resident), one row at a time.  The next row's slice of (nz_k, nz_val
// [, nz_aux]) is fetched with 16-byte cp.async.cg (L1 bypass, L2 evict-first) into the
// group's second shared-memory stage while the current row is reduced, and the next
// row's fiber columns and u_j are prefetched into registers — so the DRAM stream of row
// n+1 overlaps the gathers and arithmetic of row n.  Lane l owns the NCH consecutive
// nonzeros l·NCH .. l·NCH+NCH-1 of the row; fiber membership comes from the head flag in
// bit 31 of nz_k (per-lane bits + one exclusive scan of head counts), u_j reaches every
// nonzero by a shuffle from the lane holding its fiber, and fiber sums are a lane-serial
// pass plus one segmented scan across the group.  No block-level barriers.
//
//   r_i  = Σ_e T_e w_{k_e} u_{j_e}
//   A_f  = Σ_{e∈f} T_e w_{k_e}
//   J_f  = Σ_{e∈f} [T_e w_{k_e} + B_{i,k_e} (D_u w)_{k_e, loc(j)}]   P0 W
//   J_(i,m) = A_(i,m) + c_m Σ_{e: k_e = m} T_e u_{j_e}   W = V (IDENTITY / SQUARE)
// Per-fiber and per-row sums run in a fixed order (bitwise reproducible).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "egfem_internal.cuh"

namespace egfem {
namespace {

enum { kJacNone = 0, kJacPicard = 1, kJacNewtonWV = 2, kJacNewtonP0 = 3 };

template <typename S>
struct RowArgs {
  int64_t n_u;
  const int64_t* row_nz;
  const int64_t* row_fib;
  const int32_t* fib_j;
  const uint32_t* nz_k;
  const S* nz_val;
  const uint8_t* nz_aux;   // P0 W: cell slot of k in row i; W = V: nz_kpos
  const uint8_t* fib_kr;   // W = V: start of fiber (i, m)'s k = m run in the row's (k, j) order
  const S* u;
  const S* w;
  const S* chain;
  S* r;
  S* csr;
  int d1;
  int packed;  // P0 Newton: the gradient kinds' packed chain record [w, D_0 .. D_{d−1}], D_d = −Σ
  int dmode;   // W = V Newton factor: 0 → 1, 1 → 2u (SQUARE), 2 → −1/(pk+u)² (RECIPROCAL)
  double pk;
  uint32_t kmask;
  int64_t diag_off;  // column of row i's diagonal = i + diag_off (local tensors)
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// exact-rounding arithmetic: identical results in every template instance (no contraction choice)
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }

struct RowMeta {  // nnz < 2^32 and n_fib < 2^32 (checked at build): 32-bit offsets
  uint32_t e0, e1, f0, f1;
};
template <typename S>
__device__ __forceinline__ RowMeta row_meta(const RowArgs<S>& A, int64_t row) {
  RowMeta m{0u, 0u, 0u, 0u};
  if (row < A.n_u) {
    m.e0 = (uint32_t)__ldg(A.row_nz + row);
    m.e1 = (uint32_t)__ldg(A.row_nz + row + 1);
    m.f0 = (uint32_t)__ldg(A.row_fib + row);
    m.f1 = (uint32_t)__ldg(A.row_fib + row + 1);
  }
  return m;
}

// ---------------------------------------------------------------------------------------
// Segmented row kernel (k_seg): each lane owns NCH CONSECUTIVE nonzeros of the row
// (y = lane·NCH + c), so fibers — contiguous runs in the canonical (i, j, k) order — are
// reduced by a lane-serial pass plus one segmented scan across the G lanes (log2 G
// shuffles), with no shared-memory round trip and no divergent per-fiber loops.  The only shared-memory transposes left are the ones the algebra needs:
//   P0 W   (T·₂u)_{iK} = Σ_m T_{i v_m K} u_{v_m}: parts scattered to (cell slot, m) and
//          summed per cell (block D_zF̃ with D_u a of P0 coefficients);
//   W = V  (T·₂u)_{i m} = Σ_j T_{i j m} u_j: parts scattered to the row's (k, j) order
//          (nz_kpos) and summed per k-run (fib_kr) into fiber (i, m).
// Every sum runs in a fixed order: bitwise reproducible; the fused and separate launches
// share this code and agree bitwise.
// 16-byte async copies of the span around [p, p+n) into shared memory at 32-bit address
// dst (the address is formed once per stage, not per chunk); returns the element shift.
__device__ __forceinline__ void cp16s(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
               : "memory");
}
template <typename T, int G, int CAP>
__device__ __forceinline__ int span_copy_s(uint32_t dst, const T* p, int n, int lane, uint64_t pol) {
  constexpr int MAXCH = (CAP * (int)sizeof(T) + 31) / 16;
  constexpr int IT = (MAXCH + G - 1) / G;
  const uint64_t a = reinterpret_cast<uint64_t>(p);
  const uint64_t lo = a & ~uint64_t(15);
  const int chunks = n > 0 ? (int)((((a + (uint64_t)n * sizeof(T) + 15) & ~uint64_t(15)) - lo) >> 4) : 0;
  const char* src = reinterpret_cast<const char*>(lo) + 16 * lane;
  dst += 16 * lane;
#pragma unroll
  for (int it = 0; it < IT; ++it)
    if (lane + it * G < chunks) cp16s(dst + 16 * G * it, src + 16 * G * it, pol);
  return (int)((a - lo) / sizeof(T));
}

template <typename S, int G, int NCH, int JAC>
struct SegSmem {
  static constexpr int CAP = G * NCH;
  static constexpr bool kP0 = JAC == kJacNewtonP0;
  static constexpr bool kWV = JAC == kJacNewtonWV;
  static constexpr bool kAux = kP0 || kWV;
  static constexpr int st_k = 0;
  static constexpr int st_v = st_k + CAP * 4 + 32;
  static constexpr int st_a = st_v + CAP * (int)sizeof(S) + 32;
  static constexpr int stage = (st_a + (kAux ? CAP + 32 : 0) + 15) & ~15;
  // P0: (cell slot) x (d+1 | 1) parts of T·₂u (the row has at most CAP / (d+1) <= CAP / 3 cells)
  static constexpr int o_x = 2 * stage;
  static constexpr int o_b = o_x + (kWV ? CAP * (int)sizeof(S) : kP0 ? (CAP / 3 + 1) * 5 * (int)sizeof(S) : 0);
  // P0: B per cell; W = V: transposed sum per fiber
  static constexpr int bytes = (o_b + (kWV ? 2 * G * (int)sizeof(S) : kP0 ? (CAP / 3 + 1) * (int)sizeof(S) : 0) + 15) & ~15;
};

template <typename S, int G, int NCH, int FREG, bool DO_R, int JAC, int D1>
__global__ void __launch_bounds__(256, NCH > 8 ? 2 : ((JAC == kJacNewtonP0 || JAC == kJacNewtonWV) ? 3 : 4)) k_seg(const RowArgs<S> A) {
  using L = SegSmem<S, G, NCH, JAC>;
  constexpr int GPB = 256 / G;
  constexpr bool kP0 = L::kP0, kWV = L::kWV;
  constexpr bool kNeedU = DO_R || kP0 || kWV;
  constexpr int XS = D1 | 1;  // odd cell stride: the parts of consecutive cells spread over all banks
  // Control flow is warp-uniform (a group without a row runs on an empty one), so every
  // shuffle uses the full mask with width G.
  constexpr unsigned FM = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x % G;
  const int grp = threadIdx.x / G;
  unsigned char* gs = smem + grp * L::bytes;
  const uint32_t gs_s = smem_addr(gs);
  S* s_x = reinterpret_cast<S*>(gs + L::o_x);
  S* s_b = reinterpret_cast<S*>(gs + L::o_b);
  const uint64_t pol = l2_evict_first();
  const uint32_t KM = kP0 ? kKMask : A.kmask;  // k bits of this tensor (P0 W packs loc_j above them)
  const int64_t NG = (int64_t)gridDim.x * GPB;
  int64_t row = (int64_t)blockIdx.x * GPB + grp;
  const int64_t wrow0 = (int64_t)blockIdx.x * GPB + (threadIdx.x >> 5) * (32 / G);
  if (wrow0 >= A.n_u) return;

  // per-fiber registers: lane f holds fiber f (and f + G when FREG = 2)
  auto fibcols = [&](const RowMeta& m, int32_t* fj) {
#pragma unroll
    for (int c = 0; c < FREG; ++c) {
      const int f = lane + c * G;
      fj[c] = (kNeedU && f < (int)(m.f1 - m.f0)) ? __ldg(A.fib_j + m.f0 + f) : -1;
    }
  };
  auto ucols = [&](const int32_t* fj, S* ujl) {
#pragma unroll
    for (int c = 0; c < FREG; ++c) ujl[c] = (kNeedU && fj[c] >= 0) ? __ldg(A.u + fj[c]) : S(0);
  };
  auto stage_in = [&](uint32_t dst, const RowMeta& m, int& sk, int& sv, int& sa) {
    const int n = (int)(m.e1 - m.e0);
    sk = span_copy_s<uint32_t, G, L::CAP>(dst + L::st_k, A.nz_k + m.e0, n, lane, pol);
    sv = span_copy_s<S, G, L::CAP>(dst + L::st_v, A.nz_val + m.e0, n, lane, pol);
    sa = 0;
    if constexpr (L::kAux) sa = span_copy_s<uint8_t, G, L::CAP>(dst + L::st_a, A.nz_aux + m.e0, n, lane, pol);
  };

  RowMeta cur = row_meta(A, row);
  RowMeta nxt = row_meta(A, row + NG);
  int shk, shv, sha;
  stage_in(gs_s, cur, shk, shv, sha);
  cp_commit();
  int32_t fj_cur[FREG], fj_nxt[FREG];
  S uj_cur[FREG];
  fibcols(cur, fj_cur);
  fibcols(nxt, fj_nxt);
  ucols(fj_cur, uj_cur);
  int st = 0;
  for (int64_t wr = wrow0; wr < A.n_u; wr += NG, row += NG) {
    const int ne = (int)(cur.e1 - cur.e0);
    const int nf = (int)(cur.f1 - cur.f0);
    // ---- prefetch: metadata two rows ahead, next row's stream, u_j, fiber columns
    const RowMeta nn = row_meta(A, row + 2 * NG);
    int nshk = 0, nshv = 0, nsha = 0;
    if (row + NG < A.n_u) stage_in(gs_s + (st ^ 1) * L::stage, nxt, nshk, nshv, nsha);
    cp_commit();
    S uj_nxt[FREG];
    ucols(fj_nxt, uj_nxt);
    int32_t fj_nn[FREG];
    fibcols(nn, fj_nn);
    cp_wait1();
    __syncwarp();
    const unsigned char* cs = gs + st * L::stage;
    const int y0 = lane * NCH;
    const uint32_t* bk = reinterpret_cast<const uint32_t*>(cs + L::st_k) + shk + y0;
    const S* bv = reinterpret_cast<const S*>(cs + L::st_v) + shv + y0;
    const uint8_t* ba = reinterpret_cast<const uint8_t*>(cs + L::st_a) + sha + y0;
    const int nl = ne - y0;  // nonzeros of the row from this lane's first one on
    // ---- this lane's nonzeros, head flags, then every gather in flight together
    S tv[NCH], ww[NCH], dd[NCH];
    uint32_t kc[NCH];
    unsigned hb = 0, locs = 0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const bool ok = c < nl;
      const uint32_t k = ok ? bk[c] : 0u;
      tv[c] = ok ? bv[c] : S(0);
      if (k & kHead) hb |= 1u << c;
      ww[c] = ok ? __ldg(A.w + (k & KM)) : S(0);
      if constexpr (kP0) {
        locs |= ((k >> kKShift) & 3u) << (2 * c);
        kc[c] = k & KM;
      }
    }
    // fiber of each nonzero: heads before this lane (exclusive scan of head counts) + local
    const int hc = __popc(hb);
    int inc = hc;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      const int x = __shfl_up_sync(FM, inc, o, G);
      if (lane >= o) inc += x;
    }
    const int fbase = inc - hc - 1;  // fiber id = fbase + (heads among this lane's first c+1)
    // ---- pass 1: r, T w per nonzero, and the T·₂u parts
    S acc = S(0);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      S uj = S(0);
      if constexpr (kNeedU) {
        int fid = fbase + __popc(hb & ((2u << c) - 1u));
        fid = fid < 0 ? 0 : fid;
        const S x0 = __shfl_sync(FM, uj_cur[0], fid % G, G);
        if constexpr (FREG == 1) {
          uj = x0;
        } else {
          const S x1 = __shfl_sync(FM, uj_cur[FREG - 1], fid % G, G);
          uj = (fid < G) ? x0 : x1;
        }
      }
      const S tw = mul_(tv[c], ww[c]);
      if constexpr (DO_R) acc = fma_(tw, uj, acc);
      if constexpr (kP0) {
        if (c < nl) s_x[(int)ba[c] * XS + (int)((locs >> (2 * c)) & 3u)] = mul_(tv[c], uj);
      }
      if constexpr (kWV) {
        if (c < nl) s_x[ba[c]] = mul_(tv[c], uj);
      }
      tv[c] = tw;
    }
    if constexpr (kP0) {  // (D_u w)_{K, loc(j)}: issued here, consumed after the per-cell pass
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const uint32_t lc = (locs >> (2 * c)) & 3u;
        if (!A.packed) {
          dd[c] = (c < nl) ? __ldg(A.chain + (size_t)kc[c] * D1 + lc) : S(0);
        } else if (c < nl) {  // packed record: D_m at 1 + m, D_d = −Σ_{m<d} D_m
          const S* cr = A.chain + (size_t)kc[c] * D1;
          if (lc + 1 < (uint32_t)D1) {
            dd[c] = __ldg(cr + 1 + lc);
          } else {
            S sd = S(0);
            for (int m = 1; m < D1; ++m) sd = add_(sd, __ldg(cr + m));
            dd[c] = -sd;
          }
        } else {
          dd[c] = S(0);
        }
      }
    }
    if constexpr (DO_R) {
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) acc = add_(acc, __shfl_xor_sync(FM, acc, o, G));
      if (lane == 0 && row < A.n_u) A.r[row] = acc;
    }
    if constexpr (JAC != kJacNone) {
      if constexpr (kP0 || kWV) __syncwarp();
      if constexpr (kWV) {
        // (T·₂u)_{i m} for the fiber (i, m): its k-run in the row's (k, j) order
#pragma unroll
        for (int q = 0; q < FREG; ++q) {
          const int f = lane + q * G;
          if (f < nf) {
            const int a = __ldg(A.fib_kr + cur.f0 + f);
            const int b = (f + 1 < nf) ? (int)__ldg(A.fib_kr + cur.f0 + f + 1) : ne;
            S x = S(0);
            for (int y = a; y < b; ++y) x = add_(x, s_x[y]);
            S cm = S(1);
            if (A.dmode == 1) cm = mul_(S(2), uj_cur[q]);
            if (A.dmode == 2) {
              const S iv = S(1) / (S(A.pk) + uj_cur[q]);
              cm = -mul_(iv, iv);
            }
            s_b[f] = A.dmode ? mul_(cm, x) : x;
          }
        }
        __syncwarp();
      }
      if constexpr (kP0) {
        // (T·₂u)_{iK} per cell of the row, then t = T_ijK w_K + (T·₂u)_{iK} (D_u w)_{K, loc(j)}
        const int ncell = ne / D1;
        for (int q = lane; q < ncell; q += G) {
          S B = s_x[q * XS];
#pragma unroll
          for (int m = 1; m < D1; ++m) B = add_(B, s_x[q * XS + m]);
          s_b[q] = B;
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          if (c < nl) tv[c] = fma_(s_b[ba[c]], dd[c], tv[c]);
      }
      // ---- fiber sums: lane-serial tail, segmented inclusive scan across lanes, then each
      // fiber is finished by the lane holding its last nonzero
      S tail = S(0);
#pragma unroll
      for (int c = 0; c < NCH; ++c) tail = ((hb >> c) & 1u) ? tv[c] : add_(tail, tv[c]);
      S sv = tail;
      int fl = hb != 0;
#pragma unroll
      for (int o = 1; o < G; o <<= 1) {
        const S ov = __shfl_up_sync(FM, sv, o, G);
        const int of = __shfl_up_sync(FM, fl, o, G);
        if (lane >= o) {
          if (!fl) sv = add_(ov, sv);
          fl |= of;
        }
      }
      S run = __shfl_up_sync(FM, sv, 1, G);
      if (lane == 0) run = S(0);
      const unsigned nxh = (unsigned)__shfl_down_sync(FM, (int)(hb & 1u), 1, G);
      // bit c: nonzero c ends its fiber (the next one is a head or the row ends)
      unsigned last = (hb >> 1) | (nxh << (NCH - 1));
      if (nl >= 1 && nl <= NCH) last |= 1u << (nl - 1);
      last &= (nl >= NCH) ? ((1u << NCH) - 1u) : ((1u << (nl > 0 ? nl : 0)) - 1u);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        run = ((hb >> c) & 1u) ? tv[c] : add_(run, tv[c]);
        if ((last >> c) & 1u) {
          const int fid = fbase + __popc(hb & ((2u << c) - 1u));
          S out = run;
          if constexpr (kWV) out = add_(out, s_b[fid]);
          A.csr[cur.f0 + fid] = out;
        }
      }
    }
    __syncwarp();  // stage st and the scratch are free for reuse
    cur = nxt;
    nxt = nn;
    shk = nshk;
    shv = nshv;
    sha = nsha;
#pragma unroll
    for (int c = 0; c < FREG; ++c) {
      fj_cur[c] = fj_nxt[c];
      fj_nxt[c] = fj_nn[c];
      uj_cur[c] = uj_nxt[c];
    }
    st ^= 1;
  }
}

// W = V Newton data: per nonzero its position in the row's (k, j) order (nz_kpos) and per
// fiber (i, m) the start of the k = m run in that order (fib_kr).  Offline, one thread per row.
__global__ void k_wv_aux(int64_t n_u, const int64_t* __restrict__ row_fib, const uint32_t* __restrict__ fib_nz,
                         const int32_t* __restrict__ fib_j, const uint32_t* __restrict__ nz_k, uint8_t* kpos,
                         uint8_t* kr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_u) return;
  const int64_t f0 = row_fib[i], f1 = row_fib[i + 1];
  const uint32_t r0 = fib_nz[f0], r1 = fib_nz[f1];
  for (int64_t f = f0; f < f1; ++f) {
    const int32_t j = fib_j[f];
    uint32_t before = 0;  // nonzeros of the row with k < j
    for (uint32_t e = r0; e < r1; ++e) before += ((int32_t)(nz_k[e] & kKMaskAny) < j) ? 1u : 0u;
    kr[f] = (uint8_t)before;
    for (uint32_t e = fib_nz[f]; e < fib_nz[f + 1]; ++e) {
      const int32_t k = (int32_t)(nz_k[e] & kKMaskAny);
      uint32_t pos = 0;
      for (int64_t g = f0; g < f1; ++g) {
        const int32_t j2 = fib_j[g];
        for (uint32_t e2 = fib_nz[g]; e2 < fib_nz[g + 1]; ++e2) {
          const int32_t k2 = (int32_t)(nz_k[e2] & kKMaskAny);
          pos += (k2 < k || (k2 == k && j2 < j)) ? 1u : 0u;
        }
      }
      kpos[e] = (uint8_t)pos;
    }
  }
}

int g_sms[64] = {0};

template <typename S, int G, int NCH, int FREG, bool DO_R, int JAC, int D1 = 0>
egfem_status run_rows(const egfem_tensor* t, const RowArgs<S>& A, cudaStream_t s) {
  auto fn = k_seg<S, G, NCH, FREG, DO_R, JAC, D1>;
  const int smem = SegSmem<S, G, NCH, JAC>::bytes * (256 / G);
  if (smem > 48 * 1024) EGFEM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int dev = t->device & 63;
  if (!g_sms[dev]) EGFEM_CUDA_TRY(cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, t->device));
  int per_sm = 0;
  EGFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem));
  const int64_t need = (t->n_u + (256 / G) - 1) / (256 / G);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)std::max(per_sm, 1) * g_sms[dev]));
  fn<<<grid, 256, smem, s>>>(A);
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

template <typename S, int G, int NCH, int FREG>
egfem_status rows_mode(const egfem_tensor* t, const RowArgs<S>& A, bool do_r, int jac, cudaStream_t s) {
  if (do_r) {
    switch (jac) {
      case kJacNone: return run_rows<S, G, NCH, FREG, true, kJacNone>(t, A, s);
      case kJacPicard: return run_rows<S, G, NCH, FREG, true, kJacPicard>(t, A, s);
      case kJacNewtonWV: return run_rows<S, G, NCH, FREG, true, kJacNewtonWV>(t, A, s);
      default:
        return t->dim == 2 ? run_rows<S, G, NCH, FREG, true, kJacNewtonP0, 3>(t, A, s)
                           : run_rows<S, G, NCH, FREG, true, kJacNewtonP0, 4>(t, A, s);
    }
  }
  switch (jac) {
    case kJacPicard: return run_rows<S, G, NCH, FREG, false, kJacPicard>(t, A, s);
    case kJacNewtonWV: return run_rows<S, G, NCH, FREG, false, kJacNewtonWV>(t, A, s);
    default:
      return t->dim == 2 ? run_rows<S, G, NCH, FREG, false, kJacNewtonP0, 3>(t, A, s)
                         : run_rows<S, G, NCH, FREG, false, kJacNewtonP0, 4>(t, A, s);
  }
}

// (lanes per row, chunks per row) from the longest row; EGFEM_ROWS_CFG="G,NCH" overrides
// (experiments; ignored when the pair cannot hold the longest row).
void rows_config(const egfem_tensor* t, int* G, int* NCH) {
  static int envG = -1, envN = -1;
  if (envG < 0) {
    envG = envN = 0;
    if (const char* e = getenv("EGFEM_ROWS_CFG")) sscanf(e, "%d,%d", &envG, &envN);
  }
  const int mx = t->max_row_nnz;
  if (envG > 0 && envG * envN >= mx) {
    *G = envG;
    *NCH = envN;
    return;
  }
  if (mx <= 16) { *G = 8; *NCH = 2; }
  else if (mx <= 32) { *G = 8; *NCH = 4; }
  else if (mx <= 64) { *G = 16; *NCH = 4; }
  else if (mx <= 96) { *G = 16; *NCH = 6; }  // two rows per warp instruction
  else if (mx <= 128) { *G = 32; *NCH = 4; }
  else if (mx <= 256) { *G = 32; *NCH = 8; }
  else if (mx <= 384) { *G = 32; *NCH = 12; }  // 3D quadrature-point W (I_2: 384 per row)
  else { *G = 32; *NCH = 16; }
}

template <typename S>
egfem_status rows_dispatch(const egfem_tensor* t, bool do_r, int jac, egfem_interp_kind kind, double p, const void* u,
                           const void* w, const void* chain, void* r, void* csr, cudaStream_t s) {
  RowArgs<S> A;
  A.n_u = t->n_u;
  A.row_nz = t->row_nz;
  A.row_fib = t->row_fib;
  A.fib_j = t->fib_j;
  A.nz_k = t->nz_k;
  A.nz_val = static_cast<const S*>(t->nz_val);
  A.nz_aux = jac == kJacNewtonWV ? t->nz_kpos : t->nz_aux;
  A.fib_kr = t->fib_kr;
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
  A.diag_off = t->row_begin - t->col_begin;
  int G = 0, NCH = 0;
  rows_config(t, &G, &NCH);
  const bool f2 = t->max_row_fib > G;
#define EGFEM_RC(g, n)                                                                                        \
  if (G == g && NCH == n)                                                                                     \
    return f2 ? rows_mode<S, g, n, (g < 32 ? 2 : 1)>(t, A, do_r, jac, s)                                 \
              : rows_mode<S, g, n, 1>(t, A, do_r, jac, s);
  EGFEM_RC(8, 2)
  EGFEM_RC(8, 4)
  EGFEM_RC(16, 4)
  EGFEM_RC(16, 6)
  EGFEM_RC(32, 3)
  EGFEM_RC(32, 4)
  EGFEM_RC(32, 8)
  EGFEM_RC(32, 12)
  EGFEM_RC(32, 16)
#undef EGFEM_RC
  set_error("no row-group configuration");
  return EGFEM_ERR_UNSUPPORTED;
}

}  // namespace

bool rows_path_ok(const egfem_tensor* t, int jac) {
  if (t->row_nz == nullptr || t->max_row_nnz > kRowsMaxNnz) return false;
  if (jac == kJacNewtonWV && (t->nz_kpos == nullptr || t->fib_kr == nullptr)) return false;
  if (jac == kJacNewtonP0 && t->dim != 2 && t->dim != 3) return false;  // 1D P0 W: tile path
  int G = 0, NCH = 0;
  rows_config(t, &G, &NCH);
  return G > 0 && G * NCH >= t->max_row_nnz && t->max_row_fib <= (G < 32 ? 2 * G : G);
}

egfem_status launch_rows(const egfem_tensor* t, bool do_r, int jac, egfem_interp_kind kind, double p, const void* u,
                         const void* w, const void* chain, void* r, void* csr_vals, cudaStream_t s) {
  if (t->n_u <= 0) return EGFEM_OK;
  if (t->dtype == EGFEM_F64) return rows_dispatch<double>(t, do_r, jac, kind, p, u, w, chain, r, csr_vals, s);
  return rows_dispatch<float>(t, do_r, jac, kind, p, u, w, chain, r, csr_vals, s);
}

// Offline W = V Newton data for the row kernels (rows of at most kWVMaxNnz nonzeros).
egfem_status make_wv_aux(egfem_tensor* t) {
  if (!t->w_is_v || !t->newton_wv_ok || t->n_u <= 0 || t->max_row_nnz > kWVMaxNnz) return EGFEM_OK;
  EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->nz_kpos, std::max<int64_t>(t->nnz, 1)));
  EGFEM_CUDA_TRY(dmalloc_padded((void**)&t->fib_kr, std::max<int64_t>(t->n_fib, 1)));
  k_wv_aux<<<(int)((t->n_u + 127) / 128), 128>>>(t->n_u, t->row_fib, t->fib_nz, t->fib_j, t->nz_k, t->nz_kpos,
                                                  t->fib_kr);
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

}  // namespace egfem

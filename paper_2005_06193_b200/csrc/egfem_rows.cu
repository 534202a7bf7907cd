// Row-group kernels of libegfem.so (B200 / sm_100a): the fast path of steps (2)+(3).
//
// A group of G lanes (G = 8, 16 or 32, chosen from the longest row) walks rows
// grid-stride (the rows in flight stay one compact window, which keeps the w / D_u w
// gathers L2-resident), one row at a time.  The next row's slice of (nz_k, nz_val
// [, nz_aux]) is fetched with 16-byte cp.async.cg (L1 bypass, L2 evict-first) into the
// group's second shared-memory stage while the current row is reduced, and the next
// row's fiber columns are prefetched into registers — so the DRAM stream of row n+1
// overlaps the w/u gathers and arithmetic of row n.  Reads are lane-contiguous and
// bank-conflict free; w_k and u_j are gathered through L1/L2.  Fiber membership comes
// from the head flag in bit 31 of nz_k (ballot + popc) and u_j reaches every nonzero
// by a shuffle from the lane holding its fiber.  No block-level barriers.
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
  const uint8_t* nz_aux;
  const S* u;
  const S* w;
  const S* chain;
  S* r;
  S* csr;
  int d1;
  bool square;
  uint32_t kmask;
  int64_t diag_off;  // column of row i's diagonal = i + diag_off (local tensors)
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 16-byte async global→shared copy that bypasses L1 and is evicted first from L2.
__device__ __forceinline__ void cp16(void* dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Copy the 16-byte-aligned span around [p, p+n) (n <= CAP) into dst with a fully unrolled,
// predicated loop; returns the element shift of p inside the span.
template <typename T, int G, int CAP>
__device__ __forceinline__ int span_copy(unsigned char* dst, const T* p, int n, int lane, uint64_t pol) {
  constexpr int MAXCH = (CAP * (int)sizeof(T) + 31) / 16;
  constexpr int IT = (MAXCH + G - 1) / G;
  const uint64_t a = reinterpret_cast<uint64_t>(p);
  const uint64_t lo = a & ~uint64_t(15);
  const int chunks = n > 0 ? (int)((((a + (uint64_t)n * sizeof(T) + 15) & ~uint64_t(15)) - lo) >> 4) : 0;
  const char* src = reinterpret_cast<const char*>(lo);
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int q = lane + it * G;
    if (q < chunks) cp16(dst + 16 * q, src + 16 * q, pol);
  }
  return (int)((a - lo) / sizeof(T));
}

// exact-rounding arithmetic: identical results in every template instance (no contraction choice)
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }

template <typename S, int G, int NCH, int JAC>
struct RowSmem {  // per-group shared memory
  static constexpr int CAP = G * NCH;
  static constexpr bool kAny = JAC != kJacNone;
  static constexpr bool kP0 = JAC == kJacNewtonP0;
  static constexpr bool kWV = JAC == kJacNewtonWV;
  // double-buffered stream stages (+32 B alignment slack each)
  static constexpr int st_k = 0;
  static constexpr int st_v = st_k + CAP * 4 + 32;
  static constexpr int st_a = st_v + CAP * (int)sizeof(S) + 32;
  static constexpr int stage = (st_a + (kP0 ? CAP + 32 : 0) + 15) & ~15;
  // Jacobian scratch
  static constexpr int o_t = 2 * stage;                                     // S[CAP]  per-nonzero terms
  static constexpr int o_x = o_t + (kAny ? CAP * (int)sizeof(S) : 0);       // S[CAP]  B parts / T u_j
  static constexpr int o_b = o_x + ((kP0 || kWV) ? CAP * (int)sizeof(S) : 0);  // S[CAP] B per cell / extra per fiber
  static constexpr int o_k = o_b + ((kP0 || kWV) ? CAP * (int)sizeof(S) : 0);  // u32[CAP] k (WV)
  static constexpr int o_fs = o_k + (kWV ? CAP * 4 : 0);                    // i16[CAP+2] fiber starts
  static constexpr int bytes_raw = o_fs + (kAny ? (CAP + 2) * 2 : 0);
  static constexpr int bytes = (bytes_raw + 15) & ~15;
};

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

template <typename S, int G, int NCH, int FREG, bool DO_R, int JAC>
__global__ void __launch_bounds__(256) k_rows(const RowArgs<S> A) {
  using L = RowSmem<S, G, NCH, JAC>;
  constexpr int GPB = 256 / G;
  constexpr bool kNeedU = DO_R || JAC >= kJacNewtonWV;
  constexpr unsigned GM = (G == 32) ? 0xffffffffu : ((1u << G) - 1u);
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x % G;
  const int grp = threadIdx.x / G;
  const int wl = threadIdx.x & 31;
  const int goff = wl & ~(G - 1);
  // Control flow is warp-uniform (a group without a row runs on an empty one), so every
  // shuffle / ballot uses the full mask with width G and no divergence handling is emitted.
  constexpr unsigned gmask = 0xffffffffu;
  const unsigned lane_le = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
  unsigned char* gs = smem + grp * L::bytes;
  S* s_t = reinterpret_cast<S*>(gs + L::o_t);
  S* s_x = reinterpret_cast<S*>(gs + L::o_x);
  S* s_b = reinterpret_cast<S*>(gs + L::o_b);
  uint32_t* s_k = reinterpret_cast<uint32_t*>(gs + L::o_k);
  int16_t* s_fs = reinterpret_cast<int16_t*>(gs + L::o_fs);
  const uint64_t pol = l2_evict_first();
  // grid-stride over rows: the rows in flight form one compact window, so the w / D_u w
  // gathers of all groups hit the same L2-resident neighbourhood
  const int64_t NG = (int64_t)gridDim.x * GPB;
  int64_t row = (int64_t)blockIdx.x * GPB + grp;
  const int64_t wrow0 = (int64_t)blockIdx.x * GPB + (threadIdx.x >> 5) * (32 / G);  // first row of the warp
  if (wrow0 >= A.n_u) return;

  auto fibcols = [&](const RowMeta& m, int32_t* fj) {
#pragma unroll
    for (int c = 0; c < FREG; ++c) {
      const int f = lane + c * G;
      fj[c] = ((kNeedU || JAC != kJacNone) && f < (int)(m.f1 - m.f0)) ? __ldg(A.fib_j + m.f0 + f) : -1;
    }
  };
  auto ucols = [&](const int32_t* fj, S* ujl) {
#pragma unroll
    for (int c = 0; c < FREG; ++c) ujl[c] = (kNeedU && fj[c] >= 0) ? __ldg(A.u + fj[c]) : S(0);
  };

  RowMeta cur = row_meta(A, row);
  RowMeta nxt = row_meta(A, row + NG);
  int shk = span_copy<uint32_t, G, L::CAP>(gs + L::st_k, A.nz_k + cur.e0, (int)(cur.e1 - cur.e0), lane, pol);
  int shv = span_copy<S, G, L::CAP>(gs + L::st_v, A.nz_val + cur.e0, (int)(cur.e1 - cur.e0), lane, pol);
  int sha = 0;
  if (L::kP0) sha = span_copy<uint8_t, G, L::CAP>(gs + L::st_a, A.nz_aux + cur.e0, (int)(cur.e1 - cur.e0), lane, pol);
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
    // ---- prefetch: metadata two rows ahead, next row's stream, next row's u_j, fiber columns
    const RowMeta nn = row_meta(A, row + 2 * NG);
    int nshk = 0, nshv = 0, nsha = 0;
    if (row + NG < A.n_u) {
      unsigned char* ns = gs + (st ^ 1) * L::stage;
      const int nne = (int)(nxt.e1 - nxt.e0);
      nshk = span_copy<uint32_t, G, L::CAP>(ns + L::st_k, A.nz_k + nxt.e0, nne, lane, pol);
      nshv = span_copy<S, G, L::CAP>(ns + L::st_v, A.nz_val + nxt.e0, nne, lane, pol);
      if (L::kP0) nsha = span_copy<uint8_t, G, L::CAP>(ns + L::st_a, A.nz_aux + nxt.e0, nne, lane, pol);
    }
    cp_commit();
    S uj_nxt[FREG];
    ucols(fj_nxt, uj_nxt);
    int32_t fj_nn[FREG];
    fibcols(nn, fj_nn);
    // ---- this row's stream has landed
    cp_wait1();
    __syncwarp();
    const unsigned char* cs = gs + st * L::stage;
    const uint32_t* bk = reinterpret_cast<const uint32_t*>(cs + L::st_k) + shk;
    const S* bv = reinterpret_cast<const S*>(cs + L::st_v) + shv;
    const uint8_t* ba = reinterpret_cast<const uint8_t*>(cs + L::st_a) + sha;
    // ---- k of every chunk, then all w gathers in flight together
    uint32_t kk[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int y = lane + c * G;
      kk[c] = (y < ne) ? bk[y] : 0u;
    }
    S ww[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) ww[c] = (lane + c * G < ne) ? __ldg(A.w + (kk[c] & A.kmask)) : S(0);
    S dd[NCH];
    if constexpr (L::kP0) {
#pragma unroll
      for (int c = 0; c < NCH; ++c)
        dd[c] = (lane + c * G < ne)
                    ? __ldg(A.chain + (int64_t)(kk[c] & A.kmask) * A.d1 + ((kk[c] >> kKShift) & 3u))
                    : S(0);
    }
    // ---- pass 1 (streaming): r and the per-nonzero Jacobian parts
    S acc = S(0);
    int cnt = 0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int y = lane + c * G;
      const bool h = (y < ne) && (kk[c] & kHead);
      const unsigned hm = (__ballot_sync(gmask, h) >> goff) & GM;
      const int fid = cnt + __popc(hm & lane_le) - 1;
      cnt += __popc(hm);
      if constexpr (JAC != kJacNone) {
        if (h) s_fs[fid] = (int16_t)y;
      }
      const S vv = (y < ne) ? bv[y] : S(0);
      S uj = S(0);
      if constexpr (kNeedU) {
        const int ff = fid < 0 ? 0 : fid;
        const S x0 = __shfl_sync(gmask, uj_cur[0], ff % G, G);
        if constexpr (FREG == 1) {
          uj = x0;
        } else {
          const S x1 = __shfl_sync(gmask, uj_cur[FREG - 1], ff % G, G);
          uj = (ff < G) ? x0 : x1;
        }
      }
      const S vw = mul_(vv, ww[c]);
      if constexpr (DO_R) acc = fma_(vw, uj, acc);
      if (y < ne) {
        if constexpr (JAC == kJacPicard) s_t[y] = vw;
        if constexpr (L::kP0) {
          s_t[y] = vw;
          s_x[(int)ba[y] * A.d1 + (int)((kk[c] >> kKShift) & 3u)] = mul_(vv, uj);
        }
        if constexpr (JAC == kJacNewtonWV) {
          s_t[y] = vw;
          s_x[y] = mul_(vv, uj);
          s_k[y] = kk[c] & A.kmask;
        }
      }
    }
    if constexpr (DO_R) {
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) acc = add_(acc, __shfl_xor_sync(gmask, acc, o, G));
      if (lane == 0 && row < A.n_u) A.r[row] = acc;
    }
    if constexpr (JAC != kJacNone) {
      if (lane == 0) s_fs[nf] = (int16_t)ne;
      __syncwarp();
      if constexpr (L::kP0) {
        // (T·₂u)_{iK} = Σ_m T_{i v_m K} u_{v_m}: one lane per cell of the row sums its d+1 parts
        const int ncell = ne / A.d1;
        for (int q = lane; q < ncell; q += G) {
          S B = S(0);
          for (int m = 0; m < A.d1; ++m) B = add_(B, s_x[q * A.d1 + m]);
          s_b[q] = B;
        }
        __syncwarp();
        // t = T_ijK w_K + B_{iK} (D_u w)_{K, loc(j)}
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int y = lane + c * G;
          if (y < ne) s_t[y] = fma_(s_b[ba[y]], dd[c], s_t[y]);
        }
      }
      if constexpr (JAC == kJacNewtonWV) {
        // transposed term per fiber (i, m): c_m Σ_{(j, k=m) in row i} T_ijm u_j, in row order
        for (int f = lane; f < nf; f += G) {
          const uint32_t m = (uint32_t)__ldg(A.fib_j + cur.f0 + f);
          S a = S(0);
          for (int y = 0; y < ne; ++y)
            if (s_k[y] == m) a = add_(a, s_x[y]);
          s_b[f] = A.square ? mul_(mul_(S(2), __ldg(A.u + m)), a) : a;
        }
      }
      __syncwarp();
      // ---- fiber sums into the CSR values.  The diagonal fiber (j = i) is the long one (one
      // entry per cell around i for P0 W): the whole group sums it lane-strided + butterfly;
      // every other fiber (a few cells around an edge) is summed by one lane in order.
      const int32_t irow = (int32_t)(row + A.diag_off);
      int fd = -1;
#pragma unroll
      for (int c = 0; c < FREG; ++c) {
        const unsigned b = (__ballot_sync(gmask, fj_cur[c] == irow) >> goff) & GM;
        if (b) fd = c * G + __ffs(b) - 1;
      }
      for (int f = lane; f < nf; f += G) {
        if (f == fd) continue;
        const int ya = s_fs[f], yb = s_fs[f + 1];
        S a = S(0);
        for (int y = ya; y < yb; ++y) a = add_(a, s_t[y]);
        if constexpr (JAC == kJacNewtonWV) a = add_(a, s_b[f]);
        A.csr[cur.f0 + f] = a;
      }
      {
        const int ya = fd >= 0 ? s_fs[fd] : 0, yb = fd >= 0 ? s_fs[fd + 1] : 0;
        S a = S(0);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int y = ya + lane + c * G;
          if (y < yb) a = add_(a, s_t[y]);
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) a = add_(a, __shfl_xor_sync(gmask, a, o, G));
        if (lane == 0 && fd >= 0) {
          if constexpr (JAC == kJacNewtonWV) a = add_(a, s_b[fd]);
          A.csr[cur.f0 + fd] = a;
        }
      }
    }
    __syncwarp();  // all lanes are done with stage st (and the scratch) before reuse
    // ---- rotate
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

int g_sms[64] = {0};

template <typename S, int G, int NCH, int FREG, bool DO_R, int JAC>
egfem_status run_rows(const egfem_tensor* t, const RowArgs<S>& A, cudaStream_t s) {
  using L = RowSmem<S, G, NCH, JAC>;
  auto fn = k_rows<S, G, NCH, FREG, DO_R, JAC>;
  const int smem = L::bytes * (256 / G);
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
      default: return run_rows<S, G, NCH, FREG, true, kJacNewtonP0>(t, A, s);
    }
  }
  switch (jac) {
    case kJacPicard: return run_rows<S, G, NCH, FREG, false, kJacPicard>(t, A, s);
    case kJacNewtonWV: return run_rows<S, G, NCH, FREG, false, kJacNewtonWV>(t, A, s);
    default: return run_rows<S, G, NCH, FREG, false, kJacNewtonP0>(t, A, s);
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
  else { *G = 32; *NCH = 8; }
}

template <typename S>
egfem_status rows_dispatch(const egfem_tensor* t, bool do_r, int jac, egfem_interp_kind kind, const void* u,
                           const void* w, const void* chain, void* r, void* csr, cudaStream_t s) {
  RowArgs<S> A;
  A.n_u = t->n_u;
  A.row_nz = t->row_nz;
  A.row_fib = t->row_fib;
  A.fib_j = t->fib_j;
  A.nz_k = t->nz_k;
  A.nz_val = static_cast<const S*>(t->nz_val);
  A.nz_aux = t->nz_aux;
  A.u = static_cast<const S*>(u);
  A.w = static_cast<const S*>(w);
  A.chain = static_cast<const S*>(chain);
  A.r = static_cast<S*>(r);
  A.csr = static_cast<S*>(csr);
  A.d1 = t->dim + 1;
  A.square = kind == EGFEM_INTERP_SQUARE;
  A.kmask = t->kmask();
  A.diag_off = t->row_begin - t->col_begin;
  int G = 0, NCH = 0;
  rows_config(t, &G, &NCH);
  const bool f2 = t->max_row_fib > G;
#define EGFEM_RC(g, n)                                                                                   \
  if (G == g && NCH == n)                                                                                \
    return f2 ? rows_mode<S, g, n, (g < 32 ? 2 : 1)>(t, A, do_r, jac, s) : rows_mode<S, g, n, 1>(t, A, do_r, jac, s);
  EGFEM_RC(8, 2)
  EGFEM_RC(8, 4)
  EGFEM_RC(16, 4)
  EGFEM_RC(16, 6)
  EGFEM_RC(32, 3)
  EGFEM_RC(32, 4)
  EGFEM_RC(32, 8)
#undef EGFEM_RC
  set_error("no row-group configuration");
  return EGFEM_ERR_UNSUPPORTED;
}

}  // namespace

bool rows_path_ok(const egfem_tensor* t) {
  if (t->row_nz == nullptr || t->max_row_nnz > kRowsMaxNnz) return false;
  int G = 0, NCH = 0;
  rows_config(t, &G, &NCH);
  return G > 0 && G * NCH >= t->max_row_nnz && t->max_row_fib <= (G < 32 ? 2 * G : G);
}

egfem_status launch_rows(const egfem_tensor* t, bool do_r, int jac, egfem_interp_kind kind, const void* u,
                         const void* w, const void* chain, void* r, void* csr_vals, cudaStream_t s) {
  if (t->n_u <= 0) return EGFEM_OK;
  if (t->dtype == EGFEM_F64) return rows_dispatch<double>(t, do_r, jac, kind, u, w, chain, r, csr_vals, s);
  return rows_dispatch<float>(t, do_r, jac, kind, u, w, chain, r, csr_vals, s);
}

}  // namespace egfem

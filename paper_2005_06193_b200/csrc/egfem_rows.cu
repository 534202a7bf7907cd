// Row-group kernels of libegfem.so (B200 / sm_100a): the fast path of steps (2)+(3).
//
// One group of G lanes (G = 8, 16 or 32) owns one row i at a time (grid-stride over
// rows, consecutive groups on consecutive rows).  The row's nonzeros are read
// lane-contiguously — G·NCH of them per round, all chunk loads issued before any is
// used — with streaming (L2 evict-first) loads, so the T stream is perfectly
// coalesced and many requests are in flight per lane; w_k is gathered through L1/L2.
// Fiber membership comes from the head flag in bit 31 of nz_k (ballot + popc), so the
// hot loop never reads fib_nz.  There are no block-level barriers: groups progress
// independently and the SM interleaves their memory and compute phases.
//
//   r_i  = Σ_e T_e w_{k_e} u_{j_e}
//   A_f  = Σ_{e∈f} T_e w_{k_e}
//   J_f  = Σ_{e∈f} [T_e w_{k_e} + B_{i,k_e} (D_u w)_{k_e, loc(j)}]   P0 W
//   J_(i,m) = A_(i,m) + c_m Σ_{e: k_e = m} T_e u_{j_e}   W = V (IDENTITY / SQUARE)
// Per-fiber and per-row sums run in a fixed order (bitwise reproducible).
#include <algorithm>

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
};

__device__ __forceinline__ uint32_t ldcs_u32(const uint32_t* p) { return __ldcs(p); }
__device__ __forceinline__ double ldcs_s(const double* p) { return __ldcs(p); }
__device__ __forceinline__ float ldcs_s(const float* p) { return __ldcs(p); }

template <typename S, int G, int NCH, int JAC>
struct RowSmem {  // per-group scratch (only the Jacobian variants need any)
  static constexpr int CAP = G * NCH;
  static constexpr bool kAny = JAC != kJacNone;
  static constexpr int o_p = 0;                                          // S[CAP]  per-nonzero terms
  static constexpr int o_x = o_p + (kAny ? CAP * (int)sizeof(S) : 0);    // S[CAP]  B parts / T u_j
  static constexpr int o_k = o_x + ((JAC >= kJacNewtonWV) ? CAP * (int)sizeof(S) : 0);  // u32[CAP] k (WV)
  static constexpr int o_fs = o_k + ((JAC == kJacNewtonWV) ? CAP * 4 : 0);              // i16[CAP+1] fiber starts
  static constexpr int bytes_raw = o_fs + (kAny ? (CAP + 2) * 2 : 0);
  static constexpr int bytes = (bytes_raw + 15) & ~15;
};

template <typename S, int G, int NCH, bool DO_R, int JAC>
__global__ void __launch_bounds__(256) k_rows(const RowArgs<S> A) {
  using L = RowSmem<S, G, NCH, JAC>;
  constexpr int GPB = 256 / G;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x % G;
  const int grp = threadIdx.x / G;
  const int wl = threadIdx.x & 31;
  const int goff = wl & ~(G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << goff);
  unsigned char* gs = smem + grp * L::bytes;
  S* s_p = reinterpret_cast<S*>(gs + L::o_p);
  S* s_x = reinterpret_cast<S*>(gs + L::o_x);
  uint32_t* s_k = reinterpret_cast<uint32_t*>(gs + L::o_k);
  int16_t* s_fs = reinterpret_cast<int16_t*>(gs + L::o_fs);
  const unsigned lane_le = (G == 32 && lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);

  for (int64_t row = (int64_t)blockIdx.x * GPB + grp; row < A.n_u; row += (int64_t)gridDim.x * GPB) {
    const int64_t e0 = A.row_nz[row];
    const int ne = (int)(A.row_nz[row + 1] - e0);
    const int64_t f0 = A.row_fib[row];
    // ---- stream the row's nonzeros (all chunk loads in flight at once)
    uint32_t kk[NCH];
    S vv[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int y = lane + c * G;
      kk[c] = 0;
      vv[c] = S(0);
      if (y < ne) {
        kk[c] = ldcs_u32(A.nz_k + e0 + y);
        vv[c] = ldcs_s(A.nz_val + e0 + y);
      }
    }
    S ww[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int y = lane + c * G;
      ww[c] = (y < ne) ? __ldg(A.w + (kk[c] & A.kmask)) : S(0);
    }
    // ---- fiber index of every nonzero: running count of head flags
    int fid[NCH];
    int nf = 0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int y = lane + c * G;
      const bool h = (y < ne) && (kk[c] & kHead);
      const unsigned b = (__ballot_sync(gmask, h) >> goff) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u));
      fid[c] = nf + __popc(b & lane_le) - 1;
      if constexpr (JAC != kJacNone) {
        if (h) s_fs[fid[c]] = (int16_t)y;
      }
      nf += __popc(b);
    }
    // ---- u_j of every nonzero (fib_j and u are L1/L2 resident)
    constexpr bool kNeedU = DO_R || JAC >= kJacNewtonWV;
    S uj[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int y = lane + c * G;
      uj[c] = S(0);
      if (kNeedU && y < ne) uj[c] = __ldg(A.u + __ldg(A.fib_j + f0 + fid[c]));
    }
    if constexpr (DO_R) {
      S acc = S(0);
#pragma unroll
      for (int c = 0; c < NCH; ++c) acc += vv[c] * ww[c] * uj[c];
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gmask, acc, o, G);
      if (lane == 0) A.r[row] = acc;
    }
    if constexpr (JAC != kJacNone) {
      if (lane == 0) s_fs[nf] = (int16_t)ne;
      if constexpr (JAC == kJacNewtonP0) {
        // (T·₂u)_{iK} parts T_ijK u_j at unique slots (cell slot of K, local index of j in K)
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int y = lane + c * G;
          if (y < ne)
            s_x[(int)__ldcs(A.nz_aux + e0 + y) * A.d1 + (int)((kk[c] >> kKShift) & 3u)] = vv[c] * uj[c];
        }
        __syncwarp(gmask);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int y = lane + c * G;
          if (y < ne) {
            const uint32_t k = kk[c] & A.kmask;
            const int m = (int)((kk[c] >> kKShift) & 3u);
            const int b = (int)__ldcs(A.nz_aux + e0 + y) * A.d1;
            S B = S(0);
            for (int q = 0; q < A.d1; ++q) B += s_x[b + q];
            const S D = __ldg(A.chain + (int64_t)k * A.d1 + m);
            s_p[y] = vv[c] * ww[c] + B * D;
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int y = lane + c * G;
          if (y < ne) {
            s_p[y] = vv[c] * ww[c];
            if constexpr (JAC == kJacNewtonWV) {
              s_x[y] = vv[c] * uj[c];
              s_k[y] = kk[c] & A.kmask;
            }
          }
        }
      }
      __syncwarp(gmask);
      // ---- one lane per fiber: ordered fiber sums into the CSR values
      for (int f = lane; f < nf; f += G) {
        const int ya = s_fs[f], yb = s_fs[f + 1];
        S a = S(0);
        for (int y = ya; y < yb; ++y) a += s_p[y];
        if constexpr (JAC == kJacNewtonWV) {
          const uint32_t m = (uint32_t)__ldg(A.fib_j + f0 + f);
          S acc = S(0);
          for (int y = 0; y < ne; ++y)
            if (s_k[y] == m) acc += s_x[y];
          const S cm = A.square ? S(2) * __ldg(A.u + m) : S(1);
          a += cm * acc;
        }
        A.csr[f0 + f] = a;
      }
      __syncwarp(gmask);
    }
  }
}

int g_sms[64] = {0};

template <typename S, int G, int NCH, bool DO_R, int JAC>
egfem_status run_rows(const egfem_tensor* t, const RowArgs<S>& A, cudaStream_t s) {
  using L = RowSmem<S, G, NCH, JAC>;
  auto fn = k_rows<S, G, NCH, DO_R, JAC>;
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

template <typename S, int G, int NCH>
egfem_status rows_mode(const egfem_tensor* t, const RowArgs<S>& A, bool do_r, int jac, cudaStream_t s) {
  if (do_r) {
    switch (jac) {
      case kJacNone: return run_rows<S, G, NCH, true, kJacNone>(t, A, s);
      case kJacPicard: return run_rows<S, G, NCH, true, kJacPicard>(t, A, s);
      case kJacNewtonWV: return run_rows<S, G, NCH, true, kJacNewtonWV>(t, A, s);
      default: return run_rows<S, G, NCH, true, kJacNewtonP0>(t, A, s);
    }
  }
  switch (jac) {
    case kJacPicard: return run_rows<S, G, NCH, false, kJacPicard>(t, A, s);
    case kJacNewtonWV: return run_rows<S, G, NCH, false, kJacNewtonWV>(t, A, s);
    default: return run_rows<S, G, NCH, false, kJacNewtonP0>(t, A, s);
  }
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
  const int mx = t->max_row_nnz;
  if (mx <= 16) return rows_mode<S, 8, 2>(t, A, do_r, jac, s);
  if (mx <= 32) return rows_mode<S, 8, 4>(t, A, do_r, jac, s);
  if (mx <= 64) return rows_mode<S, 16, 4>(t, A, do_r, jac, s);
  if (mx <= 128) return rows_mode<S, 32, 4>(t, A, do_r, jac, s);
  return rows_mode<S, 32, 8>(t, A, do_r, jac, s);
}

}  // namespace

bool rows_path_ok(const egfem_tensor* t) { return t->row_nz != nullptr && t->max_row_nnz <= kRowsMaxNnz; }

egfem_status launch_rows(const egfem_tensor* t, bool do_r, int jac, egfem_interp_kind kind, const void* u,
                         const void* w, const void* chain, void* r, void* csr_vals, cudaStream_t s) {
  if (t->n_u <= 0) return EGFEM_OK;
  if (t->dtype == EGFEM_F64) return rows_dispatch<double>(t, do_r, jac, kind, u, w, chain, r, csr_vals, s);
  return rows_dispatch<float>(t, do_r, jac, kind, u, w, chain, r, csr_vals, s);
}

}  // namespace egfem

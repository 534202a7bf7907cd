// Batched tensor action (step (2b), cfg5) in a dense-local-block layout (B200 / sm_100a).
//
//   R_{i,p} = Σ_{(j,k)} T_ijk U_{j,p} W_{k,p}       for p < batch
//
// For W = V forms every nonzero of row i has j and k in the row's CSR stencil
// N(i) = {j : (i, j) fiber} (the cell cliques around i), so row i of T is a small dense
// |N|×|N| block M_i[a][b] = T_{i, N_a, N_b} (zero where T has no nonzero).  The builder keeps
// that block per row (row-major, stride |N| rounded up to even).  A warp owns 32·PPT pairs
// (lane, lane+32, …; PPT = 2) of one row at a time: it loads
// W at the stencil into registers, then
//   R_{i,p} = Σ_a U_{N_a,p} Σ_b M_i[a][b] W_{N_b,p}
// is pure FP64 FMAs with register operands and warp-uniform (broadcast) block loads, so
// each W value fetched is reused |N| times and each block value PPT times per lane — the batched
// action is FP64-bound instead of L1-gather-bound.  The per-row stencil size is a template
// parameter (dispatched per row, warp-uniform).  Fixed summation order: bitwise reproducible.
#include <algorithm>
#include <vector>

#include "egfem_internal.cuh"

namespace egfem {
namespace {

constexpr int kDenseMaxN = 20;  // longest stencil with a dense-block instance
constexpr int kDense1MaxN = 16;  // longest stencil of the single-vector dense kernel (one lane per point)
int g_sms_dense1[64] = {0};

template <typename S>
struct DenseArgs {
  int64_t n_u, n_f;
  int32_t B;
  const int64_t* row_fib;
  const int32_t* fib_j;
  const int64_t* blk_off;
  const S* blk;
  const S* U;
  const S* W;
  S* R;
};

template <bool NM>
__device__ __forceinline__ int64_t at(int64_t node, int p, int32_t B, int64_t n) {
  return NM ? node * B + p : (int64_t)p * n + node;
}

template <typename S>
struct Vec2;
template <>
struct Vec2<double> {
  using T = double2;
};
template <>
struct Vec2<float> {
  using T = float2;
};

// PPT pairs per lane (lane, lane+32, ...): each staged block value feeds PPT FMAs and each W
// value N; even and odd b accumulate in separate chains.  W at the row's stencil is loaded by
// load_w (one row ahead of its use, see k_dense).
template <typename S, int N, bool NM, int PPT>
__device__ __forceinline__ void load_w(const DenseArgs<S>& A, const int32_t* cols, int p0, S (&wv)[PPT][N]) {
#pragma unroll
  for (int b = 0; b < N; ++b) {
    const int64_t k = cols[b];  // smem broadcast
#pragma unroll
    for (int q = 0; q < PPT; ++q)
      wv[q][b] = (p0 + 32 * q < A.B) ? __ldg(A.W + at<NM>(k, p0 + 32 * q, A.B, A.n_f)) : S(0);
  }
}

template <typename S, int N, bool NM, int PPT>
__device__ __forceinline__ void dense_row(const DenseArgs<S>& A, int64_t row, const int32_t* cols, const S* M, int p0,
                                          const S (&wv)[PPT][N]) {
  constexpr int NP = N + (N & 1);
  bool ok[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) ok[q] = p0 + 32 * q < A.B;
  S r[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) r[q] = S(0);
#pragma unroll
  for (int a = 0; a < N; ++a) {
    const int64_t j = cols[a];
    S uu[PPT], se[PPT], so[PPT];
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      uu[q] = ok[q] ? __ldg(A.U + at<NM>(j, p0 + 32 * q, A.B, A.n_u)) : S(0);
      se[q] = S(0);
      so[q] = S(0);
    }
#pragma unroll
    for (int b = 0; b < N; b += 2) {
      const typename Vec2<S>::T m = *reinterpret_cast<const typename Vec2<S>::T*>(M + a * NP + b);  // smem broadcast
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        se[q] = fma(m.x, wv[q][b], se[q]);
        if (b + 1 < N) so[q] = fma(m.y, wv[q][b + 1], so[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < PPT; ++q) r[q] = fma(uu[q], se[q] + so[q], r[q]);
  }
#pragma unroll
  for (int q = 0; q < PPT; ++q)
    if (ok[q]) A.R[at<NM>(row, p0 + 32 * q, A.B, A.n_u)] = r[q];
}

__device__ __forceinline__ void cp16_dense(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// One launch per stencil width N (rows grouped by N offline, `dense_rows`, and their blocks
// stored contiguously in that order), so every instance holds exactly 2N W values per lane and
// the narrow stencils run at high occupancy.  The class's rows (listed in row order: neighbours
// share most of their stencil) are cut into batches of RB, dealt round-robin to the CTAs; a
// CTA's next batch (one contiguous span of blocks) and its stencil columns are copied into
// shared memory by cp.async while this batch is used; its warps take the 64-pair chunks of
// each row.
template <int N, typename S>
struct DenseTile {
  static constexpr int NP = N + (N & 1);
  static constexpr int RB = N > 0 ? ((2048 / (N * NP)) > 0 ? (2048 / (N * NP)) : 1) : 1;  // rows per stage
  static constexpr int BYTES = (RB * N * NP * (int)sizeof(S) + 32 + 15) & ~15;
};

template <int N>
struct DensePPT {  // pairs per lane (4 for N <= 12 measured slower on cfg5: 1.73 vs 1.53 ms)
  static constexpr int value = 2;
};

template <typename S, int N, bool NM>
__global__ void __launch_bounds__(128) k_dense(const DenseArgs<S> A, const int32_t* __restrict__ rows, int64_t nrows,
                                              int64_t blk0, int rb) {
  using TL = DenseTile<N, S>;
  constexpr int PPT = DensePPT<N>::value;
  constexpr int NP = TL::NP, RB = TL::RB;
  __shared__ __align__(16) unsigned char s_blk[2][N > 0 ? TL::BYTES : 16];
  __shared__ int32_t s_cols[2][N > 0 ? RB * N : 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int nchunks = (A.B + 32 * PPT - 1) / (32 * PPT);
  // batches of RB consecutive class entries, dealt round-robin to the CTAs: the rows in flight
  // form one moving window, so the U / W rows their stencils touch stay L2-resident
  const int64_t q1 = nrows;
  // rb <= RB rows per batch: small classes use short batches so that every SM gets work
  const int64_t step = (int64_t)gridDim.x * rb;
  const int64_t q0 = (int64_t)blockIdx.x * rb;
  if (q0 >= q1) return;
  if constexpr (N == 0) {  // empty rows
    for (int64_t q = (int64_t)blockIdx.x; q < q1; q += gridDim.x)
      for (int p = threadIdx.x; p < A.B; p += blockDim.x) A.R[at<NM>(rows[q], p, A.B, A.n_u)] = S(0);
    return;
  } else {
    // stage entries [q, min(q + RB, q1)) of the class list into buffer b; returns the shift
    auto stage = [&](int64_t q, int b) -> int {
      if (q >= q1) return 0;
      const int nr = (int)(q1 - q < (int64_t)rb ? q1 - q : (int64_t)rb);
      for (int x = threadIdx.x; x < nr * N; x += blockDim.x) {
        const int64_t row = __ldg(rows + q + x / N);
        s_cols[b][x] = __ldg(A.fib_j + __ldg(A.row_fib + row) + x % N);
      }
      const uint64_t a0 = reinterpret_cast<uint64_t>(A.blk + blk0 + q * (N * NP));
      const uint64_t lo = a0 & ~uint64_t(15);
      const int chunks = (int)((((a0 + (uint64_t)nr * N * NP * sizeof(S) + 15) & ~uint64_t(15)) - lo) >> 4);
      for (int c = threadIdx.x; c < chunks; c += blockDim.x)
        cp16_dense(&s_blk[b][16 * c], reinterpret_cast<const char*>(lo) + 16 * c);
      return (int)((a0 - lo) / sizeof(S));
    };
    int sh_cur = stage(q0, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    int st = 0;
    for (int64_t q = q0; q < q1; q += step) {
      const int sh_nxt = stage(q + step, st ^ 1);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncthreads();  // this batch's blocks and columns are in buffer st for every warp
      const int nr = (int)(q1 - q < (int64_t)rb ? q1 - q : (int64_t)rb);
      const S* M = reinterpret_cast<const S*>(s_blk[st]) + sh_cur;
      for (int ch = warp; ch < nchunks; ch += nwarps) {
        const int p0 = ch * 32 * PPT + lane;
        if constexpr (N > 12) {  // wide stencils: no register room for a second W set
          for (int r = 0; r < nr; ++r) {
            S wa[PPT][N];
            load_w<S, N, NM, PPT>(A, s_cols[st] + r * N, p0, wa);
            dense_row<S, N, NM, PPT>(A, __ldg(rows + q + r), s_cols[st] + r * N, M + r * (N * NP), p0, wa);
          }
          continue;
        }
        S wa[PPT][N], wb[PPT][N];  // W of row r (in use) and row r + 1 (in flight)
        load_w<S, N, NM, PPT>(A, s_cols[st], p0, wa);
        for (int r = 0; r < nr; r += 2) {
          if (r + 1 < nr) load_w<S, N, NM, PPT>(A, s_cols[st] + (r + 1) * N, p0, wb);
          dense_row<S, N, NM, PPT>(A, __ldg(rows + q + r), s_cols[st] + r * N, M + r * (N * NP), p0, wa);
          if (r + 1 < nr) {
            if (r + 2 < nr) load_w<S, N, NM, PPT>(A, s_cols[st] + (r + 2) * N, p0, wa);
            dense_row<S, N, NM, PPT>(A, __ldg(rows + q + r + 1), s_cols[st] + (r + 1) * N, M + (r + 1) * (N * NP), p0,
                                     wb);
          }
        }
      }
      __syncthreads();  // every warp is done with buffer st before it is refilled
      sh_cur = sh_nxt;
      st ^= 1;
    }
  }
}

// Rows outside the compiled group classes (egfem_group.cu): one warp per (row, 64-pair chunk)
// over an explicit row list of one stencil width, blocks read in place through blk_off.
template <typename S, int N>
__global__ void __launch_bounds__(128) k_dense_list(const DenseArgs<S> A, const int32_t* __restrict__ rows,
                                                   int64_t count) {
  constexpr int PPT = DensePPT<N>::value;
  constexpr int NP = N + (N & 1);
  const int lane = threadIdx.x & 31;
  const int nch = (A.B + 32 * PPT - 1) / (32 * PPT);
  const int64_t nitem = count * nch;
  const int64_t ws = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t it = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < nitem; it += ws) {
    const int64_t q = it / nch;
    const int p0 = (int)(it - q * nch) * 32 * PPT + lane;
    const int64_t row = __ldg(rows + q);
    if constexpr (N == 0) {
      for (int x = 0; x < PPT; ++x)
        if (p0 + 32 * x < A.B) A.R[at<true>(row, p0 + 32 * x, A.B, A.n_u)] = S(0);
    } else {
      const int32_t* cols = A.fib_j + __ldg(A.row_fib + row);
      const S* M = A.blk + __ldg(A.blk_off + row);
      S wa[PPT][N];
      load_w<S, N, true, PPT>(A, cols, p0, wa);
      dense_row<S, N, true, PPT>(A, row, cols, M, p0, wa);
    }
    (void)NP;
  }
}

// ------------------------------------------------------------------ single-vector W = V path
// Steps (2)+(3) for W = V tensors from the same dense blocks:
//   X_a = Σ_b M_i[a][b] w_{N_b}            Picard value of CSR slot (i, N_a)   (T·w)
//   r_i = Σ_a u_{N_a} X_a                   residual                            (T:(u⊗w))
//   Y_c = Σ_a u_{N_a} M_i[a][c]             (T·₂u)_{i N_c}
//   J_{i N_c} = X_c + f'(u_{N_c}) Y_c      Newton (f' = 1, 2u, −1/(k+u)²)
// A group of G lanes per row (rows in row order, grid-stride; a row range [lo, hi) is a
// sub-range of it): lane a owns stencil point N_a — it reads block row a (the group's reads
// cover the block contiguously), takes w_{N_b} from the other lanes by shuffles, and Y by a
// reduce-scatter of u_a M[a][·] over the group; r by a butterfly.  Fixed summation orders
// (sequential in b, fixed trees over lanes): bitwise reproducible, fused == separate.
template <typename S>
struct Dense1Args {
  const int64_t* row_fib;
  const int32_t* fib_j;
  const int64_t* blk_off;
  const S* blk;
  const S* u;
  const S* w;
  S* r;
  S* csr;
  int dmode;
  double pk;
  int64_t lo, hi;
  const S* blks;  // JAC 3: the symmetrized blocks M + Mᵀ
};

__device__ __forceinline__ double dmul1(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float dmul1(float a, float b) { return __fmul_rn(a, b); }

// JAC 3: the IDENTITY Newton with u == w (the Burgers residual is the quadratic form
// r_i = Σ_{j,k} T_ijk u_j u_k): J_ij = Σ_k T_ijk u_k + Σ_k T_ikj u_k = Σ_b (M + Mᵀ)[a][b] u_b is one
// block-row product per stencil point (no reduce-scatter for T·₂u) and r_i = ½ Σ_a u_a J_ia.
template <typename S, int G, bool DO_R, int JAC>
__global__ void __launch_bounds__(256) k_dense1(const Dense1Args<S> A) {
  constexpr bool kN = JAC == 2;  // W = V Newton
  constexpr bool kS = JAC == 3;  // W = V IDENTITY Newton, u == w, symmetrized blocks
  constexpr bool kU = DO_R || kN || kS;
  constexpr unsigned FM = 0xffffffffu;
  constexpr int RPW = 32 / G;  // rows per warp
  const int lane = threadIdx.x % G;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x / G);
  // warp-uniform loop: a group past the end runs on an empty row.  Software-pipelined: the next
  // row's (f0, n, block offset) are loaded during the current row and its stencil column one
  // step behind them, so the u / w gathers and block reads of a row are the only loads it waits on.
  struct Meta1 {
    int64_t f0;
    int n;
    int64_t off;
  };
  auto meta = [&](int64_t row) {
    Meta1 x{0, 0, 0};
    if (row < A.hi) {
      x.f0 = __ldg(A.row_fib + row);
      x.n = (int)(__ldg(A.row_fib + row + 1) - x.f0);
      x.off = __ldg(A.blk_off + row);
    }
    return x;
  };
  const int64_t wr0 = A.lo + ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / G;
  const int64_t gofs = (threadIdx.x & 31) / G;
  Meta1 cur = meta(wr0 + gofs);
  Meta1 nxt = meta(wr0 + gofs + stride);
  int jc = lane < cur.n ? __ldg(A.fib_j + cur.f0 + lane) : 0;
  for (int64_t wr = wr0; wr < A.hi; wr += stride) {
    const int64_t row = wr + gofs;
    const bool live = row < A.hi;
    const Meta1 nn = meta(row + 2 * stride);
    const int jn = lane < nxt.n ? __ldg(A.fib_j + nxt.f0 + lane) : 0;
    const int n = cur.n;
    const int64_t f0 = cur.f0;
    const int np = n + (n & 1);
    const S* M = (kS ? A.blks : A.blk) + cur.off;
    const bool has = lane < n;
    const S wl = __ldg(A.w + jc);  // j = 0 for lanes past the stencil: a valid, unused value
    const S ul = kU ? __ldg(A.u + jc) : S(0);
    // block row `lane` (16-byte loads) and column `lane`
    S m[G + 1], c[G];
#pragma unroll
    for (int b = 0; b < G; b += 2) {
      if (has && b < n) {
        const typename Vec2<S>::T v = __ldg(reinterpret_cast<const typename Vec2<S>::T*>(M + lane * np + b));
        m[b] = v.x;
        m[b + 1] = v.y;
      } else {
        m[b] = S(0);
        m[b + 1] = S(0);
      }
    }
    S X = S(0), Y = S(0);
#pragma unroll
    for (int b = 0; b < G; ++b) {
      const S wb = __shfl_sync(FM, wl, b, G);
      if (b < n) X = fma(m[b], wb, X);
    }
    if constexpr (kN) {
      // Y_l = Σ_a u_a M[a][l]: lane a forms u_a M[a][·] from its own row, then a fixed-tree
      // reduce-scatter over the group leaves component l in lane l
#pragma unroll
      for (int l = 0; l < G; ++l) c[l] = has ? dmul1(ul, m[l]) : S(0);
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int t = 0; t < o; ++t) {
          const S send = upper ? c[t] : c[t + o];
          const S keep = upper ? c[t + o] : c[t];
          c[t] = keep + __shfl_xor_sync(FM, send, o, G);
        }
      }
      Y = c[0];
    }
    if constexpr (DO_R) {
      S acc = has ? dmul1(ul, X) : S(0);
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) acc = acc + __shfl_xor_sync(FM, acc, o, G);
      if (live && lane == 0) A.r[row] = kS ? dmul1(S(0.5), acc) : acc;
    }
    if constexpr (JAC != 0) {
      if (has) {
        S v = X;
        if constexpr (kN) {
          S cm = S(1);
          if (A.dmode == 1) cm = dmul1(S(2), ul);
          if (A.dmode == 2) {
            const S iv = S(1) / (S(A.pk) + ul);
            cm = -dmul1(iv, iv);
          }
          v = A.dmode ? fma(cm, Y, v) : v + Y;
        }
        A.csr[f0 + lane] = v;
      }
    }
    cur = nxt;
    nxt = nn;
    jc = jn;
  }
  (void)RPW;
}

template <typename S, int NMAX, bool DO_R, int JAC>
egfem_status run_dense1(const egfem_tensor* t, const Dense1Args<S>& A, cudaStream_t s) {
  auto fn = k_dense1<S, NMAX, DO_R, JAC>;
  const int dev = t->device & 63;
  int per_sm = 0;
  EGFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
  const int64_t need = (A.hi - A.lo + (256 / NMAX) - 1) / (256 / NMAX);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)std::max(per_sm, 1) * g_sms_dense1[dev]));
  fn<<<grid, 256, 0, s>>>(A);
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

template <typename S, int NMAX>
egfem_status dense1_mode(const egfem_tensor* t, const Dense1Args<S>& A, bool do_r, int jac, cudaStream_t s) {
  if (do_r) {
    if (jac == 3) return run_dense1<S, NMAX, true, 3>(t, A, s);
    if (jac == 0) return run_dense1<S, NMAX, true, 0>(t, A, s);
    if (jac == 1) return run_dense1<S, NMAX, true, 1>(t, A, s);
    return run_dense1<S, NMAX, true, 2>(t, A, s);
  }
  if (jac == 1) return run_dense1<S, NMAX, false, 1>(t, A, s);
  return run_dense1<S, NMAX, false, 2>(t, A, s);
}

template <typename S>
egfem_status dense1_dispatch(const egfem_tensor* t, int64_t lo, int64_t hi, bool do_r, int jac,
                             egfem_interp_kind kind, double p, const void* u, const void* w, void* r, void* csr,
                             cudaStream_t s) {
  Dense1Args<S> A{t->row_fib, t->fib_j, t->blk_off, static_cast<const S*>(t->blk), static_cast<const S*>(u),
                  static_cast<const S*>(w), static_cast<S*>(r), static_cast<S*>(csr),
                  kind == EGFEM_INTERP_SQUARE ? 1 : (kind == EGFEM_INTERP_RECIPROCAL ? 2 : 0), p, lo, hi,
                  static_cast<const S*>(t->blk_sym)};
  // the fused IDENTITY Newton with u and w the same array: the symmetrized blocks (k_dense1 JAC 3)
  static int sym_env = -1;
  if (sym_env < 0) sym_env = getenv("EGFEM_DENSE_SYM") ? (atoi(getenv("EGFEM_DENSE_SYM")) != 0) : 1;
  if (do_r && jac == 2 && kind == EGFEM_INTERP_IDENTITY && u == w && t->blk_sym && sym_env) jac = 3;
  const int dev = t->device & 63;
  if (!g_sms_dense1[dev])
    EGFEM_CUDA_TRY(cudaDeviceGetAttribute(&g_sms_dense1[dev], cudaDevAttrMultiProcessorCount, t->device));
  const int mx = t->max_row_fib;  // G lanes per row, one per stencil point
  if (mx <= 4) return dense1_mode<S, 4>(t, A, do_r, jac, s);
  if (mx <= 8) return dense1_mode<S, 8>(t, A, do_r, jac, s);
  return dense1_mode<S, 16>(t, A, do_r, jac, s);
}

// Offline: the dense block of each row (one thread per row).  err = 1 if a k lies outside
// its row's stencil (then the tensor keeps only the CSF kernels).
template <typename S>
__global__ void k_make_dense(int64_t n_u, const int64_t* __restrict__ row_fib, const int32_t* __restrict__ fib_j,
                             const uint32_t* __restrict__ fib_nz, const uint32_t* __restrict__ nz_k,
                             const S* __restrict__ nz_val, const int64_t* __restrict__ blk_off, S* blk, int* err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_u) return;
  const int64_t f0 = row_fib[i], f1 = row_fib[i + 1];
  const int n = (int)(f1 - f0);
  const int np = n + (n & 1);
  S* M = blk + blk_off[i];
  for (int x = 0; x < n * np; ++x) M[x] = S(0);
  for (int64_t f = f0; f < f1; ++f)
    for (uint32_t e = fib_nz[f]; e < fib_nz[f + 1]; ++e) {
      const int32_t k = (int32_t)(nz_k[e] & kKMaskAny);
      int lo = 0, hi = n;
      while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (fib_j[f0 + mid] < k) lo = mid + 1; else hi = mid;
      }
      if (lo >= n || fib_j[f0 + lo] != k) {
        atomicExch(err, 1);
        return;
      }
      M[(f - f0) * np + lo] = nz_val[e];
    }
}

// Offline: M + Mᵀ of each row's block (W = V; the IDENTITY Newton of k_dense1 JAC 3).
template <typename S>
__global__ void k_make_dense_sym(int64_t n_u, const int64_t* __restrict__ row_fib, const int64_t* __restrict__ blk_off,
                                 const S* __restrict__ blk, S* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_u) return;
  const int n = (int)(row_fib[i + 1] - row_fib[i]);
  const int np = n + (n & 1);
  const S* M = blk + blk_off[i];
  S* O = out + blk_off[i];
  for (int a = 0; a < n; ++a) {
    for (int b = 0; b < n; ++b) O[a * np + b] = M[a * np + b] + M[b * np + a];
    if (np > n) O[a * np + n] = S(0);
  }
}

int g_sms_dense[64] = {0};

}  // namespace

bool dense_path_ok(const egfem_tensor* t) { return t->blk != nullptr; }

// single vector: W = V tensors with dense blocks and stencils of at most 16 (jac: 0 none,
// 1 Picard, 2 W = V Newton)
bool dense1_path_ok(const egfem_tensor* t, int jac) {
  return t->blk != nullptr && t->w_is_v && t->max_row_fib <= kDense1MaxN && jac >= 0 && jac <= 2;
}

egfem_status launch_dense1(const egfem_tensor* t, int64_t lo, int64_t hi, bool do_r, int jac, egfem_interp_kind kind,
                           double p, const void* u, const void* w, void* r, void* csr_vals, cudaStream_t s) {
  if (hi <= lo) return EGFEM_OK;
  if (t->dtype == EGFEM_F64) return dense1_dispatch<double>(t, lo, hi, do_r, jac, kind, p, u, w, r, csr_vals, s);
  return dense1_dispatch<float>(t, lo, hi, do_r, jac, kind, p, u, w, r, csr_vals, s);
}

egfem_status launch_dense(const egfem_tensor* t, int32_t batch, egfem_layout layout, const void* U, const void* W,
                          void* R, cudaStream_t s) {
  if (t->n_u <= 0) return EGFEM_OK;
  const int dev = t->device & 63;
  if (!g_sms_dense[dev])
    EGFEM_CUDA_TRY(cudaDeviceGetAttribute(&g_sms_dense[dev], cudaDevAttrMultiProcessorCount, t->device));
  const bool nm = layout == EGFEM_LAYOUT_NODE_MAJOR;
  // one launch per stencil width; each a single wave of resident CTAs over its row list
  for (const auto& cls : t->dense_classes) {
    const int n = (int)cls[0];
    const int64_t start = cls[1], count = cls[2];
    const int32_t* rows = t->dense_rows + start;
#define EGFEM_DN(S_, N_)                                                                                       \
  case N_: {                                                                                                  \
    DenseArgs<S_> A{t->n_u, t->n_f, batch, t->row_fib, t->fib_j, t->blk_off, (const S_*)t->blk,              \
                    (const S_*)U, (const S_*)W, (S_*)R};                                                      \
    auto fn = nm ? k_dense<S_, N_, true> : k_dense<S_, N_, false>;                                            \
    const int threads = 32 * std::min(4, (batch + 32 * DensePPT<N_>::value - 1) / (32 * DensePPT<N_>::value)); \
    int per_sm = 0;                                                                                           \
    EGFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0));                   \
    const int64_t slots = (int64_t)std::max(per_sm, 1) * g_sms_dense[dev];                                   \
    const int rb = (int)std::max<int64_t>(1, std::min<int64_t>(DenseTile<N_, S_>::RB, (count + slots - 1) / slots)); \
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((count + rb - 1) / rb, slots));               \
    fn<<<grid, threads, 0, s>>>(A, rows, count, cls[3], rb);                                                  \
    break;                                                                                                    \
  }
#define EGFEM_DALL(S_)                                                                                         \
  switch (n) {                                                                                                \
    EGFEM_DN(S_, 0) EGFEM_DN(S_, 1) EGFEM_DN(S_, 2) EGFEM_DN(S_, 3) EGFEM_DN(S_, 4) EGFEM_DN(S_, 5)          \
    EGFEM_DN(S_, 6) EGFEM_DN(S_, 7) EGFEM_DN(S_, 8) EGFEM_DN(S_, 9) EGFEM_DN(S_, 10) EGFEM_DN(S_, 11)        \
    EGFEM_DN(S_, 12) EGFEM_DN(S_, 13) EGFEM_DN(S_, 14) EGFEM_DN(S_, 15) EGFEM_DN(S_, 16) EGFEM_DN(S_, 17)   \
    EGFEM_DN(S_, 18) EGFEM_DN(S_, 19) EGFEM_DN(S_, 20)                                                        \
    default: set_error("dense stencil wider than 20"); return EGFEM_ERR_UNSUPPORTED;                         \
  }
    if (t->dtype == EGFEM_F64) {
      EGFEM_DALL(double)
    } else {
      EGFEM_DALL(float)
    }
#undef EGFEM_DALL
#undef EGFEM_DN
    count_launch();
  }
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

egfem_status launch_dense_rows(const egfem_tensor* t, int32_t batch, const int32_t* rows,
                               const std::vector<std::array<int64_t, 3>>& classes, const void* U, const void* W,
                               void* R, cudaStream_t s) {
  const int dev = t->device & 63;
  if (!g_sms_dense[dev])
    EGFEM_CUDA_TRY(cudaDeviceGetAttribute(&g_sms_dense[dev], cudaDevAttrMultiProcessorCount, t->device));
  for (const auto& cls : classes) {
    const int n = (int)cls[0];
    const int64_t start = cls[1], count = cls[2];
    const int nch = (batch + 63) / 64;
    const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>((count * nch + 3) / 4, (int64_t)g_sms_dense[dev] * 16));
#define EGFEM_DL(S_, N_)                                                                                  \
  case N_: {                                                                                             \
    DenseArgs<S_> A{t->n_u, t->n_f, batch, t->row_fib, t->fib_j, t->blk_off, (const S_*)t->blk,         \
                    (const S_*)U, (const S_*)W, (S_*)R};                                                 \
    k_dense_list<S_, N_><<<(unsigned)ctas, 128, 0, s>>>(A, rows + start, count);                         \
    break;                                                                                               \
  }
#define EGFEM_DLALL(S_)                                                                                   \
  switch (n) {                                                                                           \
    EGFEM_DL(S_, 0) EGFEM_DL(S_, 1) EGFEM_DL(S_, 2) EGFEM_DL(S_, 3) EGFEM_DL(S_, 4) EGFEM_DL(S_, 5)     \
    EGFEM_DL(S_, 6) EGFEM_DL(S_, 7) EGFEM_DL(S_, 8) EGFEM_DL(S_, 9) EGFEM_DL(S_, 10) EGFEM_DL(S_, 11)   \
    EGFEM_DL(S_, 12) EGFEM_DL(S_, 13) EGFEM_DL(S_, 14) EGFEM_DL(S_, 15) EGFEM_DL(S_, 16) EGFEM_DL(S_, 17) \
    EGFEM_DL(S_, 18) EGFEM_DL(S_, 19) EGFEM_DL(S_, 20)                                                   \
    default: set_error("dense stencil wider than 20"); return EGFEM_ERR_UNSUPPORTED;                    \
  }
    if (t->dtype == EGFEM_F64) {
      EGFEM_DLALL(double)
    } else {
      EGFEM_DLALL(float)
    }
#undef EGFEM_DLALL
#undef EGFEM_DL
    count_launch();
  }
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

// Offline dense blocks for W = V tensors whose stencils are at most kDenseMaxN wide.
egfem_status make_dense_blocks(egfem_tensor* t, const std::vector<int64_t>& hrf) {
  if (!t->w_is_v || t->n_u <= 0 || t->nnz <= 0 || t->max_row_fib > kDenseMaxN) return EGFEM_OK;
  // rows grouped by stencil width (stable: row order within a width); blocks stored in that order
  std::vector<int32_t> order(t->n_u);
  std::vector<int64_t> cnt(kDenseMaxN + 2, 0);
  for (int64_t i = 0; i < t->n_u; ++i) cnt[hrf[i + 1] - hrf[i] + 1]++;
  for (int n = 0; n <= kDenseMaxN; ++n) cnt[n + 1] += cnt[n];
  std::vector<int64_t> first(cnt.begin(), cnt.end() - 1);
  for (int64_t i = 0; i < t->n_u; ++i) order[first[hrf[i + 1] - hrf[i]]++] = (int32_t)i;
  std::vector<int64_t> off(t->n_u + 1, 0);  // off[i]: block of row i; off[n_u]: total
  int64_t pos = 0;
  t->dense_classes.clear();
  for (int n = 0; n <= kDenseMaxN; ++n) {
    if (cnt[n + 1] == cnt[n]) continue;
    t->dense_classes.push_back({n, cnt[n], cnt[n + 1] - cnt[n], pos});
    for (int64_t q = cnt[n]; q < cnt[n + 1]; ++q) {
      off[order[q]] = pos;
      pos += (int64_t)n * (n + (n & 1));
    }
  }
  off[t->n_u] = pos;
  const size_t vs = t->dtype == EGFEM_F64 ? 8 : 4;
  EGFEM_CUDA_TRY(cudaMalloc(&t->blk_off, 8 * (t->n_u + 1)));
  EGFEM_CUDA_TRY(cudaMemcpy(t->blk_off, off.data(), 8 * (t->n_u + 1), cudaMemcpyHostToDevice));
  EGFEM_CUDA_TRY(dmalloc_padded(&t->blk, vs * std::max<int64_t>(off[t->n_u], 1)));
  int* err = nullptr;
  EGFEM_CUDA_TRY(cudaMalloc(&err, sizeof(int)));
  EGFEM_CUDA_TRY(cudaMemset(err, 0, sizeof(int)));
  const int nb = (int)((t->n_u + 127) / 128);
  if (t->dtype == EGFEM_F64)
    k_make_dense<double><<<nb, 128>>>(t->n_u, t->row_fib, t->fib_j, t->fib_nz, t->nz_k, (const double*)t->nz_val,
                                      t->blk_off, (double*)t->blk, err);
  else
    k_make_dense<float><<<nb, 128>>>(t->n_u, t->row_fib, t->fib_j, t->fib_nz, t->nz_k, (const float*)t->nz_val,
                                     t->blk_off, (float*)t->blk, err);
  count_launch();
  int herr = 0;
  cudaError_t ce = cudaMemcpy(&herr, err, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(err);
  EGFEM_CUDA_TRY(ce);
  if (herr) {
    cudaFree(t->blk_off);
    cudaFree(t->blk);
    t->blk_off = nullptr;
    t->blk = nullptr;
    t->dense_classes.clear();
    return EGFEM_OK;
  }
  EGFEM_CUDA_TRY(cudaMalloc(&t->dense_rows, sizeof(int32_t) * t->n_u));
  EGFEM_CUDA_TRY(cudaMemcpy(t->dense_rows, order.data(), sizeof(int32_t) * t->n_u, cudaMemcpyHostToDevice));
  // the symmetrized blocks for the single-vector IDENTITY Newton with u == w (stencils <= 16)
  if (t->max_row_fib <= kDense1MaxN) {
    EGFEM_CUDA_TRY(dmalloc_padded(&t->blk_sym, vs * std::max<int64_t>(off[t->n_u], 1)));
    if (t->dtype == EGFEM_F64)
      k_make_dense_sym<double><<<nb, 128>>>(t->n_u, t->row_fib, t->blk_off, (const double*)t->blk, (double*)t->blk_sym);
    else
      k_make_dense_sym<float><<<nb, 128>>>(t->n_u, t->row_fib, t->blk_off, (const float*)t->blk, (float*)t->blk_sym);
    count_launch();
    EGFEM_CUDA_TRY(cudaGetLastError());
  }
  return EGFEM_OK;
}

}  // namespace egfem

// Batched tensor action (step (2b), cfg5) in a dense-local-block layout (B200 / sm_100a).
//
//   R_{i,p} = Σ_{(j,k)} T_ijk U_{j,p} W_{k,p}       for p < batch
//
// For W = V forms every nonzero of row i has j and k in the row's CSR stencil
// N(i) = {j : (i, j) fiber} (the cell cliques around i), so row i of T is a small dense
// |N|×|N| block M_i[a][b] = T_{i, N_a, N_b} (zero where T has no nonzero).  The builder keeps
// that block per row (row-major, stride |N| rounded up to even).  A warp owns 64 pairs
// (lane, lane+32) of one row at a time: it loads W at the stencil into registers, then
//   R_{i,p} = Σ_a U_{N_a,p} Σ_b M_i[a][b] W_{N_b,p}
// is pure FP64 FMAs with register operands and warp-uniform (broadcast) block loads, so
// each W value fetched is reused |N| times and each block value 2× per lane — the batched
// action is FP64-bound instead of L1-gather-bound.  The per-row stencil size is a template
// parameter (dispatched per row, warp-uniform).  Fixed summation order: bitwise reproducible.
#include <algorithm>
#include <vector>

#include "egfem_internal.cuh"

namespace egfem {
namespace {

constexpr int kDenseMaxN = 20;  // longest stencil with a dense-block instance

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

template <typename S, int N, bool NM>
__device__ __forceinline__ void dense_row(const DenseArgs<S>& A, int64_t row, const int32_t* cols, const S* M, int p0) {
  constexpr int NP = N + (N & 1);
  const int p1 = p0 + 32;
  const bool ok0 = p0 < A.B, ok1 = p1 < A.B;
  S w0[N], w1[N];
#pragma unroll
  for (int b = 0; b < N; ++b) {
    const int64_t k = cols[b];  // smem broadcast
    w0[b] = ok0 ? __ldg(A.W + at<NM>(k, p0, A.B, A.n_f)) : S(0);
    w1[b] = ok1 ? __ldg(A.W + at<NM>(k, p1, A.B, A.n_f)) : S(0);
  }
  S r0 = S(0), r1 = S(0);
#pragma unroll
  for (int a = 0; a < N; ++a) {
    const int64_t j = cols[a];
    const S u0 = ok0 ? __ldg(A.U + at<NM>(j, p0, A.B, A.n_u)) : S(0);
    const S u1 = ok1 ? __ldg(A.U + at<NM>(j, p1, A.B, A.n_u)) : S(0);
    // even and odd b in separate chains: four independent FMA chains per lane
    S s0 = S(0), s1 = S(0), t0 = S(0), t1 = S(0);
#pragma unroll
    for (int b = 0; b < N; b += 2) {
      const typename Vec2<S>::T m = *reinterpret_cast<const typename Vec2<S>::T*>(M + a * NP + b);  // smem broadcast
      s0 = fma(m.x, w0[b], s0);
      s1 = fma(m.x, w1[b], s1);
      if (b + 1 < N) {
        t0 = fma(m.y, w0[b + 1], t0);
        t1 = fma(m.y, w1[b + 1], t1);
      }
    }
    r0 = fma(u0, s0 + t0, r0);
    r1 = fma(u1, s1 + t1, r1);
  }
  if (ok0) A.R[at<NM>(row, p0, A.B, A.n_u)] = r0;
  if (ok1) A.R[at<NM>(row, p1, A.B, A.n_u)] = r1;
}

__device__ __forceinline__ void cp16_dense(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

constexpr int kBlkBytes = (kDenseMaxN * (kDenseMaxN + 1) * 8 + 32 + 15) & ~15;  // one staged block (+ slack)

// CTA c walks the contiguous rows [c·R, (c+1)·R) in order (neighbouring rows share most of
// their stencil: U/W lines are reused from L1); its warps take the 64-pair chunks of each
// row.  The next row's block is copied into shared memory (cp.async) while this one is used.
template <typename S, bool NM>
__global__ void __launch_bounds__(128) k_dense(const DenseArgs<S> A) {
  __shared__ __align__(16) unsigned char s_blk[2][kBlkBytes];
  __shared__ int32_t s_cols[2][kDenseMaxN];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int nchunks = (A.B + 63) / 64;
  const int64_t per = (A.n_u + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per;
  const int64_t r1 = min(A.n_u, r0 + per);
  if (r0 >= r1) return;
  // copy row `row`'s block (16-byte aligned span) into buffer b; returns the element shift
  auto stage = [&](int64_t row, int b) -> int {
    if (row >= r1) return 0;
    {  // the row's stencil columns (plain loads: at most kDenseMaxN, written before the barrier)
      const int64_t f0 = __ldg(A.row_fib + row), f1 = __ldg(A.row_fib + row + 1);
      for (int x = threadIdx.x; x < (int)(f1 - f0); x += blockDim.x) s_cols[b][x] = __ldg(A.fib_j + f0 + x);
    }
    const int64_t o0 = __ldg(A.blk_off + row), o1 = __ldg(A.blk_off + row + 1);
    const uint64_t a0 = reinterpret_cast<uint64_t>(A.blk + o0), a1 = reinterpret_cast<uint64_t>(A.blk + o1);
    const uint64_t lo = a0 & ~uint64_t(15);
    const int chunks = (int)((((a1 + 15) & ~uint64_t(15)) - lo) >> 4);
    for (int q = threadIdx.x; q < chunks; q += blockDim.x)
      cp16_dense(&s_blk[b][16 * q], reinterpret_cast<const char*>(lo) + 16 * q);
    return (int)((a0 - lo) / sizeof(S));
  };
  int sh_cur = stage(r0, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  int st = 0;
  for (int64_t row = r0; row < r1; ++row) {
    const int sh_nxt = stage(row + 1, st ^ 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();  // this row's block is in s_blk[st] for every warp
    const int n = (int)(__ldg(A.row_fib + row + 1) - __ldg(A.row_fib + row));
    const S* M = reinterpret_cast<const S*>(s_blk[st]) + sh_cur;
    const int32_t* cols = s_cols[st];
    for (int ch = warp; ch < nchunks; ch += nwarps) {
      const int p0 = ch * 64 + lane;
      switch (n) {
#define EGFEM_DR(N_) \
  case N_: dense_row<S, N_, NM>(A, row, cols, M, p0); break;
        EGFEM_DR(1) EGFEM_DR(2) EGFEM_DR(3) EGFEM_DR(4) EGFEM_DR(5) EGFEM_DR(6) EGFEM_DR(7) EGFEM_DR(8)
        EGFEM_DR(9) EGFEM_DR(10) EGFEM_DR(11) EGFEM_DR(12) EGFEM_DR(13) EGFEM_DR(14) EGFEM_DR(15)
        EGFEM_DR(16) EGFEM_DR(17) EGFEM_DR(18) EGFEM_DR(19) EGFEM_DR(20)
#undef EGFEM_DR
        default:  // empty row
          if (p0 < A.B) A.R[at<NM>(row, p0, A.B, A.n_u)] = S(0);
          if (p0 + 32 < A.B) A.R[at<NM>(row, p0 + 32, A.B, A.n_u)] = S(0);
      }
    }
    __syncthreads();  // every warp is done with s_blk[st] before it is refilled
    sh_cur = sh_nxt;
    st ^= 1;
  }
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

int g_sms_dense[64] = {0};

}  // namespace

bool dense_path_ok(const egfem_tensor* t) { return t->blk != nullptr; }

egfem_status launch_dense(const egfem_tensor* t, int32_t batch, egfem_layout layout, const void* U, const void* W,
                          void* R, cudaStream_t s) {
  if (t->n_u <= 0) return EGFEM_OK;
  const int dev = t->device & 63;
  if (!g_sms_dense[dev])
    EGFEM_CUDA_TRY(cudaDeviceGetAttribute(&g_sms_dense[dev], cudaDevAttrMultiProcessorCount, t->device));
  const int chunks = (batch + 63) / 64;
  const int threads = 32 * std::min(4, chunks);
  const bool nm = layout == EGFEM_LAYOUT_NODE_MAJOR;
  // one wave of resident CTAs, each walking a contiguous block of rows
#define EGFEM_D(S_)                                                                                      \
  {                                                                                                     \
    DenseArgs<S_> A{t->n_u, t->n_f, batch, t->row_fib, t->fib_j, t->blk_off, (const S_*)t->blk,        \
                    (const S_*)U, (const S_*)W, (S_*)R};                                                \
    auto fn = nm ? k_dense<S_, true> : k_dense<S_, false>;                                              \
    int per_sm = 0;                                                                                     \
    EGFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0));             \
    const int grid = (int)std::min<int64_t>(t->n_u, (int64_t)std::max(per_sm, 1) * g_sms_dense[dev]);  \
    fn<<<grid, threads, 0, s>>>(A);                                                                     \
  }
  if (t->dtype == EGFEM_F64) EGFEM_D(double) else EGFEM_D(float)
#undef EGFEM_D
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

// Offline dense blocks for W = V tensors whose stencils are at most kDenseMaxN wide.
egfem_status make_dense_blocks(egfem_tensor* t, const std::vector<int64_t>& hrf) {
  if (!t->w_is_v || t->n_u <= 0 || t->nnz <= 0 || t->max_row_fib > kDenseMaxN) return EGFEM_OK;
  std::vector<int64_t> off(t->n_u + 1, 0);
  for (int64_t i = 0; i < t->n_u; ++i) {
    const int64_t n = hrf[i + 1] - hrf[i];
    off[i + 1] = off[i] + n * (n + (n & 1));
  }
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
  }
  return EGFEM_OK;
}

}  // namespace egfem

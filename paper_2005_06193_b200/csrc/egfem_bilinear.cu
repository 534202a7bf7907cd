// Bilinear GFEM forms of libegfem.so:
// B = T·₂1 on the tensor's CSR pattern, r = B f (CSR SpMV), J = B·diag(f'(u)).
//
// The SpMV is HBM-bound (values 8 B + column 4 B per slot, x gathered): groups of G = 8 lanes
// own a row (grid-stride, so the rows in flight form one window and the x gathers stay in L2),
// lane-strided over the row's slots, reduced by a butterfly in a fixed order.
#include <algorithm>

#include "egfem_internal.cuh"

namespace egfem {
namespace {

template <typename S>
__global__ void __launch_bounds__(256) k_spmv(int64_t n_u, const int64_t* __restrict__ row_ptr,
                                              const int32_t* __restrict__ col, const S* __restrict__ vals,
                                              const S* __restrict__ x, S* __restrict__ y) {
  constexpr int G = 8;
  const int lane = threadIdx.x % G;
  const int64_t NG = (int64_t)gridDim.x * (blockDim.x / G);
  const int64_t wrow0 = (int64_t)blockIdx.x * (blockDim.x / G) + (threadIdx.x >> 5) * (32 / G);
  for (int64_t wr = wrow0, row = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G; wr < n_u;
       wr += NG, row += NG) {
    S acc = S(0);
    if (row < n_u) {
      const int64_t a = __ldg(row_ptr + row), b = __ldg(row_ptr + row + 1);
      for (int64_t q = a + lane; q < b; q += G) acc = fma(__ldcs(vals + q), __ldg(x + __ldg(col + q)), acc);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
    if (lane == 0 && row < n_u) y[row] = acc;
  }
}

// J_slot = B_slot · f'(u_col): 0 identity, 1 square (2u), 2 reciprocal (−1/(p+u)²)
template <typename S>
__global__ void k_scale_cols(int64_t nnz, const int32_t* __restrict__ col, const S* __restrict__ b,
                             const S* __restrict__ u, S* __restrict__ J, int mode, double pk) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += stride) {
    const S x = __ldg(u + __ldg(col + q));
    S d = S(1);
    if (mode == 1) d = S(2) * x;
    if (mode == 2) {
      const S iv = S(1) / (S(pk) + x);
      d = -(iv * iv);
    }
    J[q] = mode == 0 ? b[q] : b[q] * d;
  }
}

__global__ void k_fill(double* a, int64_t n, double v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}
__global__ void k_fillf(float* a, int64_t n, float v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

int g_sms_bl[64] = {0};

}  // namespace

egfem_status launch_spmv(const egfem_tensor* t, const void* vals, const void* x, void* y, cudaStream_t s) {
  if (t->n_u <= 0) return EGFEM_OK;
  const int dev = t->device & 63;
  if (!g_sms_bl[dev]) EGFEM_CUDA_TRY(cudaDeviceGetAttribute(&g_sms_bl[dev], cudaDevAttrMultiProcessorCount, t->device));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((t->n_u + 31) / 32, (int64_t)g_sms_bl[dev] * 8));
  if (t->dtype == EGFEM_F64)
    k_spmv<double><<<grid, 256, 0, s>>>(t->n_u, t->row_fib, t->fib_j, (const double*)vals, (const double*)x,
                                        (double*)y);
  else
    k_spmv<float><<<grid, 256, 0, s>>>(t->n_u, t->row_fib, t->fib_j, (const float*)vals, (const float*)x, (float*)y);
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

egfem_status launch_scale_cols(const egfem_tensor* t, const void* b, int mode, double p, const void* u, void* J,
                               cudaStream_t s) {
  if (t->n_fib <= 0) return EGFEM_OK;
  const int grid = (int)std::min<int64_t>((t->n_fib + 255) / 256, 148 * 16);
  if (t->dtype == EGFEM_F64)
    k_scale_cols<double><<<grid, 256, 0, s>>>(t->n_fib, t->fib_j, (const double*)b, (const double*)u, (double*)J,
                                              mode, p);
  else
    k_scale_cols<float><<<grid, 256, 0, s>>>(t->n_fib, t->fib_j, (const float*)b, (const float*)u, (float*)J, mode,
                                             p);
  count_launch();
  EGFEM_CUDA_TRY(cudaGetLastError());
  return EGFEM_OK;
}

// B = T·₂1: the IDENTITY Newton Jacobian T·w + T·₂u at w = 0, u = 1.
// The ones / zeros vectors span the column space (max(n_u, n_f)) and are stream-ordered
// allocations (cudaMallocAsync / cudaFreeAsync), so the call neither synchronizes nor breaks a
// CUDA-graph capture.
egfem_status launch_bilinear_build(const egfem_tensor* t, void* b_vals, cudaStream_t s) {
  const size_t vs = t->dtype == EGFEM_F64 ? 8 : 4;
  const int64_t ncol = std::max<int64_t>(std::max<int64_t>(t->n_u, t->n_f), 1);
  void* ones = nullptr;
  void* zeros = nullptr;
  EGFEM_CUDA_TRY(cudaMallocAsync(&ones, vs * ncol, s));
  if (cudaMallocAsync(&zeros, vs * ncol, s) != cudaSuccess) {
    cudaFreeAsync(ones, s);
    set_error("cudaMallocAsync failed");
    return EGFEM_ERR_OUT_OF_MEMORY;
  }
  cudaMemsetAsync(zeros, 0, vs * ncol, s);
  const int nb = (int)((ncol + 255) / 256);
  if (t->dtype == EGFEM_F64) k_fill<<<nb, 256, 0, s>>>((double*)ones, ncol, 1.0);
  else k_fillf<<<nb, 256, 0, s>>>((float*)ones, ncol, 1.0f);
  count_launch();
  egfem_status st = launch_tile(t, false, 2, EGFEM_INTERP_IDENTITY, 0.0, ones, zeros, nullptr, nullptr, b_vals, s);
  cudaFreeAsync(ones, s);
  cudaFreeAsync(zeros, s);
  return st;
}

}  // namespace egfem

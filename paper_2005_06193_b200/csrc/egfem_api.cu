// C ABI of libegfem.so: validation, handle lifetime, dispatch, multi-GPU
// partitioning.  See include/egfem.h for the contract of every entry point.
#include <nvtx3/nvToolsExt.h>
#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "egfem_internal.cuh"

namespace egfem {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

// Switch to the handle's device for the duration of a call.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

egfem_status fail(egfem_status s, const std::string& msg) {
  set_error(msg);
  return s;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Caller device pointers must be on the handle's device (or managed).
egfem_status check_dev_ptr(const egfem_tensor* t, const void* p, const char* name, bool required) {
  if (!p) return required ? fail(EGFEM_ERR_INVALID_ARGUMENT, std::string(name) + " is NULL") : EGFEM_OK;
  if (!aligned16(p)) return fail(EGFEM_ERR_INVALID_ARGUMENT, std::string(name) + " is not 16-byte aligned");
  const uintptr_t key = reinterpret_cast<uintptr_t>(p);
  {
    std::lock_guard<std::mutex> lk(t->ptr_mu);
    for (uintptr_t q : t->ptr_ok)
      if (q == key) return EGFEM_OK;
  }
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return fail(EGFEM_ERR_INVALID_ARGUMENT, std::string(name) + " is not a CUDA pointer");
  }
  if (a.type != cudaMemoryTypeManaged && (a.type != cudaMemoryTypeDevice || a.device != t->device))
    return fail(EGFEM_ERR_INVALID_ARGUMENT, std::string(name) + " is not device memory on the handle's device");
  std::lock_guard<std::mutex> lk(t->ptr_mu);
  t->ptr_ok[t->ptr_ok_next] = key;
  t->ptr_ok_next = (t->ptr_ok_next + 1) % 16;
  return EGFEM_OK;
}

egfem_status validate_space(const egfem_mesh* m, const egfem_space* S, const char* name) {
  if (!S) return fail(EGFEM_ERR_INVALID_ARGUMENT, std::string(name) + " is NULL");
  if (S->family < EGFEM_P0 || S->family > EGFEM_QUAD)
    return fail(EGFEM_ERR_INVALID_ARGUMENT, std::string(name) + ": bad family");
  if (S->family == EGFEM_QUAD) {  // N_q points per cell, each DOF used once
    if (S->n_dofs <= 0 || S->n_dofs % m->n_cells != 0 || S->n_dofs / m->n_cells > kMaxQuad)
      return fail(EGFEM_ERR_DIMENSION_MISMATCH, std::string(name) + ": QUAD needs n_dofs = N_q·n_cells, N_q <= 16");
    if (S->n_dofs >= (int64_t(1) << 31)) return fail(EGFEM_ERR_INDEX_OVERFLOW, std::string(name) + ": n_dofs");
    if (S->cell_dofs) {
      std::vector<uint8_t> seen(S->n_dofs, 0);
      for (int64_t q = 0; q < S->n_dofs; ++q) {
        if (S->cell_dofs[q] < 0 || S->cell_dofs[q] >= S->n_dofs || seen[S->cell_dofs[q]])
          return fail(EGFEM_ERR_INVALID_ARGUMENT, "QUAD cell_dofs is not a permutation");
        seen[S->cell_dofs[q]] = 1;
      }
    }
    return EGFEM_OK;
  }
  if (S->family == EGFEM_P2 && m->dim != 2) return fail(EGFEM_ERR_UNSUPPORTED, "P2 is implemented in 2D only");
  if (S->family == EGFEM_P2 && !S->cell_dofs) return fail(EGFEM_ERR_INVALID_ARGUMENT, "P2 needs cell_dofs");
  if (S->n_dofs <= 0 || S->n_dofs >= (int64_t(1) << 31))
    return fail(S->n_dofs <= 0 ? EGFEM_ERR_INVALID_ARGUMENT : EGFEM_ERR_INDEX_OVERFLOW,
                std::string(name) + ": n_dofs out of range");
  const int nl = S->family == EGFEM_P0 ? 1 : (S->family == EGFEM_P1 ? m->dim + 1 : 6);
  if (S->cell_dofs) {
    const int64_t n = m->n_cells * nl;
    for (int64_t q = 0; q < n; ++q)
      if (S->cell_dofs[q] < 0 || S->cell_dofs[q] >= S->n_dofs)
        return fail(EGFEM_ERR_INVALID_ARGUMENT, std::string(name) + ": cell_dofs entry out of range");
  } else {
    if (S->family == EGFEM_P0 && S->n_dofs != m->n_cells)
      return fail(EGFEM_ERR_DIMENSION_MISMATCH, std::string(name) + ": canonical P0 needs n_dofs == n_cells");
    if (S->family == EGFEM_P1 && S->n_dofs != m->n_vertices)
      return fail(EGFEM_ERR_DIMENSION_MISMATCH, std::string(name) + ": canonical P1 needs n_dofs == n_vertices");
  }
  if (S->family == EGFEM_P0) {  // one DOF per cell, each used once
    if (S->n_dofs != m->n_cells) return fail(EGFEM_ERR_DIMENSION_MISMATCH, "P0 needs n_dofs == n_cells");
    if (S->cell_dofs) {
      std::vector<uint8_t> seen(S->n_dofs, 0);
      for (int64_t c = 0; c < m->n_cells; ++c) {
        if (seen[S->cell_dofs[c]]) return fail(EGFEM_ERR_INVALID_ARGUMENT, "P0 cell_dofs is not a permutation");
        seen[S->cell_dofs[c]] = 1;
      }
    }
  }
  return EGFEM_OK;
}

}  // namespace

// NVTX range around an API call (SURVEY §5 tracing): header-only nvtx3, a no-op pointer check
// when no tool is attached; host-side only, so it is legal inside stream capture.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

}  // namespace egfem

using namespace egfem;

extern "C" {

const char* egfem_status_string(egfem_status s) {
  switch (s) {
    case EGFEM_OK: return "EGFEM_OK";
    case EGFEM_ERR_INVALID_ARGUMENT: return "EGFEM_ERR_INVALID_ARGUMENT";
    case EGFEM_ERR_DIMENSION_MISMATCH: return "EGFEM_ERR_DIMENSION_MISMATCH";
    case EGFEM_ERR_UNSUPPORTED: return "EGFEM_ERR_UNSUPPORTED";
    case EGFEM_ERR_INDEX_OVERFLOW: return "EGFEM_ERR_INDEX_OVERFLOW";
    case EGFEM_ERR_OUT_OF_MEMORY: return "EGFEM_ERR_OUT_OF_MEMORY";
    case EGFEM_ERR_CUDA: return "EGFEM_ERR_CUDA";
    case EGFEM_ERR_NCCL: return "EGFEM_ERR_NCCL";
  }
  return "EGFEM_UNKNOWN";
}

const char* egfem_last_error(void) { return g_last_error.c_str(); }

uint64_t egfem_launch_count(void) { return g_launches.load(); }

egfem_status egfem_tensor_build(const egfem_mesh* mesh, const egfem_space* V, const egfem_space* W, egfem_form form,
                                const egfem_quad* quad, egfem_dtype dtype, int device, egfem_tensor** out) {
  if (!out) return fail(EGFEM_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!mesh || !mesh->coords || !mesh->cells) return fail(EGFEM_ERR_INVALID_ARGUMENT, "mesh arrays are NULL");
  if (mesh->dim < 1 || mesh->dim > 3) return fail(EGFEM_ERR_INVALID_ARGUMENT, "dim must be 1, 2 or 3");
  if (mesh->n_cells <= 0 || mesh->n_vertices <= 0) return fail(EGFEM_ERR_INVALID_ARGUMENT, "empty mesh");
  if (mesh->n_vertices >= (int64_t(1) << 31) || mesh->n_cells >= (int64_t(1) << 31))
    return fail(EGFEM_ERR_INDEX_OVERFLOW, "mesh larger than int32 indices");
  if (form < EGFEM_FORM_CONV_K || form > EGFEM_FORM_CONV_I) return fail(EGFEM_ERR_INVALID_ARGUMENT, "bad form");
  if (dtype != EGFEM_F64 && dtype != EGFEM_F32) return fail(EGFEM_ERR_INVALID_ARGUMENT, "bad dtype");
  const int64_t ncv = mesh->n_cells * (mesh->dim + 1);
  for (int64_t q = 0; q < ncv; ++q)
    if (mesh->cells[q] < 0 || mesh->cells[q] >= mesh->n_vertices)
      return fail(EGFEM_ERR_INVALID_ARGUMENT, "mesh cell vertex out of range");
  egfem_status st = validate_space(mesh, V, "V");
  if (st) return st;
  if ((st = validate_space(mesh, W, "W"))) return st;
  if (V->family == EGFEM_P0 || V->family == EGFEM_QUAD)
    return fail(EGFEM_ERR_UNSUPPORTED, "V must be P1 or P2");
  if (W->family == EGFEM_QUAD && form == EGFEM_FORM_CONV_K)
    return fail(EGFEM_ERR_UNSUPPORTED, "QUAD W needs a value k-slot (CONV_K differentiates k)");
  if (W->family == EGFEM_QUAD && quad && quad->n_points > 0 && quad->n_points != W->n_dofs / mesh->n_cells)
    return fail(EGFEM_ERR_DIMENSION_MISMATCH, "QUAD W: quad->n_points != n_dofs / n_cells");
  if (form == EGFEM_FORM_PLAP && W->family == EGFEM_P2)
    ;  // allowed: quadrature definition
  if (quad && quad->n_points > 0 && (!quad->bary || !quad->weights))
    return fail(EGFEM_ERR_INVALID_ARGUMENT, "quadrature arrays are NULL");
  const int nV = V->family == EGFEM_P1 ? mesh->dim + 1 : 6;
  const int nW = W->family == EGFEM_P0 ? 1
                 : W->family == EGFEM_P1 ? mesh->dim + 1
                 : W->family == EGFEM_QUAD ? (int)(W->n_dofs / mesh->n_cells) : 6;
  if (nV * nV * nW > 256) return fail(EGFEM_ERR_UNSUPPORTED, "local tensor larger than 256 entries");
  if ((int64_t)nV * nV * nW * mesh->n_cells >= (int64_t(1) << 32))
    return fail(EGFEM_ERR_INDEX_OVERFLOW, "more than 2^32 element triples");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return fail(EGFEM_ERR_INVALID_ARGUMENT, "no such CUDA device");
  }
  NvtxRange nv("egfem_tensor_build");
  DeviceGuard g(device);
  if (!g.ok) return fail(EGFEM_ERR_CUDA, "cudaSetDevice failed");
  egfem_tensor* t = new egfem_tensor();
  t->device = device;
  t->dtype = dtype;
  t->form = form;
  st = upload_mesh(t, mesh, V, W);
  int64_t m = 0;
  uint64_t* key = nullptr;
  uint32_t* k = nullptr;
  double* val = nullptr;
  if (!st) st = emit_element_triples(t, form, quad, &m, &key, &k, &val);
  if (!st) {
    st = build_from_triples(t, m, key, k, val);  // takes ownership of key/k/val
  } else {
    if (key) cudaFree(key);
    if (k) cudaFree(k);
    if (val) cudaFree(val);
  }
  if (st) {
    free_tensor(t);
    delete t;
    return st;
  }
  *out = t;
  return EGFEM_OK;
}

egfem_status egfem_tensor_from_coo(int64_t n_u, int64_t n_f, int64_t nnz, const int32_t* i, const int32_t* j,
                                   const int32_t* k, const double* val, egfem_dtype dtype, int device,
                                   egfem_tensor** out) {
  if (!out) return fail(EGFEM_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (n_u <= 0 || n_f <= 0 || nnz < 0) return fail(EGFEM_ERR_INVALID_ARGUMENT, "bad sizes");
  if (n_u >= (int64_t(1) << 31) || n_f >= (int64_t(1) << 31) || nnz >= (int64_t(1) << 32))
    return fail(EGFEM_ERR_INDEX_OVERFLOW, "sizes exceed index widths");
  if (nnz > 0 && (!i || !j || !k || !val)) return fail(EGFEM_ERR_INVALID_ARGUMENT, "COO arrays are NULL");
  if (dtype != EGFEM_F64 && dtype != EGFEM_F32) return fail(EGFEM_ERR_INVALID_ARGUMENT, "bad dtype");
  std::vector<uint64_t> key(nnz);
  std::vector<uint32_t> kk(nnz);
  for (int64_t e = 0; e < nnz; ++e) {
    if (i[e] < 0 || i[e] >= n_u || j[e] < 0 || j[e] >= n_u || k[e] < 0 || k[e] >= n_f)
      return fail(EGFEM_ERR_INVALID_ARGUMENT, "COO index out of range");
    key[e] = (uint64_t)i[e] * (uint64_t)n_u + (uint64_t)j[e];
    kk[e] = (uint32_t)k[e];
  }
  bool closed = (n_u == n_f);  // T·₂u lands inside the (i,j) fiber pattern?
  if (closed) {
    std::vector<uint64_t> pat(key);
    std::sort(pat.begin(), pat.end());
    for (int64_t e = 0; e < nnz && closed; ++e)
      closed = std::binary_search(pat.begin(), pat.end(), (uint64_t)i[e] * (uint64_t)n_u + (uint64_t)k[e]);
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return fail(EGFEM_ERR_INVALID_ARGUMENT, "no such CUDA device");
  }
  NvtxRange nv("egfem_tensor_from_coo");
  DeviceGuard g(device);
  egfem_tensor* t = new egfem_tensor();
  t->device = device;
  t->dtype = dtype;
  t->n_u = n_u;
  t->n_f = n_f;
  t->w_is_v = (n_u == n_f);
  t->newton_wv_ok = closed;
  uint64_t* dkey = nullptr;
  uint32_t* dk = nullptr;
  double* dval = nullptr;
  auto cleanup = [&](egfem_status s) {
    if (dkey) cudaFree(dkey);
    if (dk) cudaFree(dk);
    if (dval) cudaFree(dval);
    free_tensor(t);
    delete t;
    return s;
  };
  const size_t n1 = (size_t)std::max<int64_t>(nnz, 1);
  if (cudaMalloc(&dkey, 8 * n1) || cudaMalloc(&dk, 4 * n1) || cudaMalloc(&dval, 8 * n1))
    return cleanup(fail(EGFEM_ERR_OUT_OF_MEMORY, "cudaMalloc failed"));
  if (nnz > 0 && (cudaMemcpy(dkey, key.data(), 8 * nnz, cudaMemcpyHostToDevice) ||
                  cudaMemcpy(dk, kk.data(), 4 * nnz, cudaMemcpyHostToDevice) ||
                  cudaMemcpy(dval, val, 8 * nnz, cudaMemcpyHostToDevice)))
    return cleanup(fail(EGFEM_ERR_CUDA, "cudaMemcpy failed"));
  egfem_status st = build_from_triples(t, nnz, dkey, dk, dval);
  dkey = nullptr;
  dk = nullptr;
  dval = nullptr;
  if (st) return cleanup(st);
  *out = t;
  return EGFEM_OK;
}

egfem_status egfem_tensor_destroy(egfem_tensor* t) {
  if (!t) return EGFEM_OK;
  NvtxRange nv("egfem_tensor_destroy");
  DeviceGuard g(t->device);
  free_tensor(t);
  delete t;
  return EGFEM_OK;
}

egfem_status egfem_tensor_info(const egfem_tensor* t, int64_t* n_u, int64_t* n_f, int64_t* nnz, int64_t* nnz_csr,
                               egfem_dtype* dtype) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  if (n_u) *n_u = t->n_u;
  if (n_f) *n_f = t->n_f;
  if (nnz) *nnz = t->nnz;
  if (nnz_csr) *nnz_csr = t->n_fib;
  if (dtype) *dtype = t->dtype;
  return EGFEM_OK;
}

egfem_status egfem_tensor_csr_pattern(const egfem_tensor* t, const int64_t** d_row_ptr, const int32_t** d_col) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  if (d_row_ptr) *d_row_ptr = t->row_fib;
  if (d_col) *d_col = t->fib_j;
  return EGFEM_OK;
}

egfem_status egfem_tensor_export(const egfem_tensor* t, int64_t* t_row_ptr, int32_t* t_j, int32_t* t_k, void* t_val,
                                 int64_t* csr_row_ptr, int32_t* csr_col, int32_t* slot_ij, int32_t* slot_ik,
                                 uint8_t* loc) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  if (slot_ik && !t->w_is_v) return fail(EGFEM_ERR_UNSUPPORTED, "slot_ik needs W = V numbering");
  if (loc && !(t->has_mesh && t->w_p0)) return fail(EGFEM_ERR_UNSUPPORTED, "loc needs W = P0");
  NvtxRange nv("egfem_tensor_export");
  DeviceGuard g(t->device);
  return export_arrays(t, t_row_ptr, t_j, t_k, t_val, csr_row_ptr, csr_col, slot_ij, slot_ik, loc);
}

static egfem_status interp_check(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u,
                                 const void* w, const void* chain) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  if (kind < EGFEM_INTERP_IDENTITY || kind > EGFEM_INTERP_RECIPROCAL)
    return fail(EGFEM_ERR_INVALID_ARGUMENT, "bad interp kind");
  egfem_status st;
  // the packed kinds hold w_k in chain[k(d+1)] too: w may then be NULL (written once, in the record)
  const bool w_opt = chain && packed_chain_kind(kind);
  if ((st = check_dev_ptr(t, u, "u", true)) || (st = check_dev_ptr(t, w, "w", !w_opt)) ||
      (st = check_dev_ptr(t, chain, "chain", false)))
    return st;
  switch (kind) {
    case EGFEM_INTERP_IDENTITY:
    case EGFEM_INTERP_SQUARE:
      if (kind == EGFEM_INTERP_SQUARE && t->wfam == EGFEM_QUAD) {  // u_h(x_ℓ)² at the quadrature points
        if (t->vfam != EGFEM_P1) return fail(EGFEM_ERR_UNSUPPORTED, "SQUARE on QUAD W needs V = P1");
        break;
      }
      if (!t->w_is_v) return fail(EGFEM_ERR_DIMENSION_MISMATCH, "IDENTITY/SQUARE need W = V (SQUARE: or QUAD)");
      if (chain) return fail(EGFEM_ERR_INVALID_ARGUMENT, "chain is only produced for cell-wise W");
      break;
    case EGFEM_INTERP_GRADPOW_P0:
      if (!t->has_mesh || !t->w_p0 || t->vfam != EGFEM_P1)
        return fail(EGFEM_ERR_UNSUPPORTED, "GRADPOW_P0 needs V = P1, W = P0 and a mesh");
      if (!(p > 1.0)) return fail(EGFEM_ERR_INVALID_ARGUMENT, "GRADPOW_P0 needs p > 1");
      break;
    case EGFEM_INTERP_MINSURF_P0:
      if (!t->has_mesh || !t->w_p0 || t->vfam != EGFEM_P1)
        return fail(EGFEM_ERR_UNSUPPORTED, "MINSURF_P0 needs V = P1, W = P0 and a mesh");
      break;
    case EGFEM_INTERP_RECIPROCAL:
      if (t->w_is_v) {
        if (chain) return fail(EGFEM_ERR_INVALID_ARGUMENT, "chain is only produced for P0 W");
      } else if (!t->has_mesh || !t->w_p0 || t->vfam != EGFEM_P1) {
        return fail(EGFEM_ERR_UNSUPPORTED, "RECIPROCAL needs W = V, or V = P1 and W = P0 with a mesh");
      }
      if (!std::isfinite(p)) return fail(EGFEM_ERR_INVALID_ARGUMENT, "RECIPROCAL needs a finite p (= k)");
      break;
    default:
      if (!t->has_mesh || t->vfam != EGFEM_P1 || t->wfam != EGFEM_P2 || t->dim != 2)
        return fail(EGFEM_ERR_UNSUPPORTED, "P1_TO_P2_SQUARE needs V = P1, W = P2 (2D)");
      if (chain) return fail(EGFEM_ERR_INVALID_ARGUMENT, "chain is only produced by GRADPOW_P0");
  }
  return EGFEM_OK;
}

egfem_status egfem_interp(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u, void* w,
                          void* chain, egfem_stream_t stream) {
  egfem_status st = interp_check(t, kind, p, u, w, chain);
  if (st) return st;
  NvtxRange nv("egfem_interp");
  DeviceGuard g(t->device);
  return launch_interp(t, kind, p, u, w, chain, 0, interp_items(t, kind), (cudaStream_t)stream);
}

egfem_status egfem_interp_range(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u, void* w,
                                void* chain, int64_t lo, int64_t hi, egfem_stream_t stream) {
  egfem_status st = interp_check(t, kind, p, u, w, chain);
  if (st) return st;
  if (lo < 0 || hi < lo || hi > interp_items(t, kind))
    return fail(EGFEM_ERR_INVALID_ARGUMENT, "interp range outside [0, n_items]");
  NvtxRange nv("egfem_interp_range");
  DeviceGuard g(t->device);
  return launch_interp(t, kind, p, u, w, chain, lo, hi, (cudaStream_t)stream);
}

egfem_status egfem_apply(const egfem_tensor* t, const void* u, const void* w, void* r, egfem_stream_t stream) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  egfem_status st;
  if ((st = check_dev_ptr(t, u, "u", true)) || (st = check_dev_ptr(t, w, "w", true)) ||
      (st = check_dev_ptr(t, r, "r", true)))
    return st;
  NvtxRange nv("egfem_apply");
  DeviceGuard g(t->device);
  return launch_tile(t, true, 0, EGFEM_INTERP_IDENTITY, 0.0, u, w, nullptr, r, nullptr, (cudaStream_t)stream);
}

egfem_status egfem_apply_batched(const egfem_tensor* t, int32_t batch, egfem_layout layout, const void* U,
                                 const void* W, void* R, egfem_stream_t stream) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  if (batch < 1) return fail(EGFEM_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (layout != EGFEM_LAYOUT_NODE_MAJOR && layout != EGFEM_LAYOUT_PAIR_MAJOR)
    return fail(EGFEM_ERR_INVALID_ARGUMENT, "bad layout");
  if ((int64_t)batch * std::max(t->n_u, t->n_f) >= (int64_t(1) << 62))
    return fail(EGFEM_ERR_INDEX_OVERFLOW, "batch too large");
  egfem_status st;
  if ((st = check_dev_ptr(t, U, "U", true)) || (st = check_dev_ptr(t, W, "W", true)) ||
      (st = check_dev_ptr(t, R, "R", true)))
    return st;
  NvtxRange nv("egfem_apply_batched");
  DeviceGuard g(t->device);
  return launch_batched(t, batch, layout, U, W, R, (cudaStream_t)stream);
}

static egfem_status jac_mode_code(const egfem_tensor* t, egfem_jac_mode mode, egfem_interp_kind kind, double p,
                                  const void* u, const void* chain, int* code, bool check_ptrs = true) {
  if (mode == EGFEM_JAC_PICARD) {
    *code = 1;
    return EGFEM_OK;
  }
  if (mode != EGFEM_JAC_NEWTON) return fail(EGFEM_ERR_INVALID_ARGUMENT, "bad Jacobian mode");
  egfem_status st;
  if (check_ptrs && (st = check_dev_ptr(t, u, "u", true))) return st;
  switch (kind) {
    case EGFEM_INTERP_IDENTITY:
    case EGFEM_INTERP_SQUARE:
      if (kind == EGFEM_INTERP_SQUARE && t->wfam == EGFEM_QUAD && t->vfam == EGFEM_P1) {
        if (check_ptrs && (st = check_dev_ptr(t, chain, "chain", true))) return st;
        *code = 3;
        return EGFEM_OK;
      }
      if (!t->w_is_v) return fail(EGFEM_ERR_DIMENSION_MISMATCH, "IDENTITY/SQUARE Newton needs W = V");
      if (!t->newton_wv_ok)
        return fail(EGFEM_ERR_UNSUPPORTED, "T·₂u has entries outside the CSR pattern (from_coo tensor)");
      *code = 2;
      return EGFEM_OK;
    case EGFEM_INTERP_GRADPOW_P0:
    case EGFEM_INTERP_MINSURF_P0:
      if (!t->has_mesh || !t->w_p0 || t->vfam != EGFEM_P1)
        return fail(EGFEM_ERR_UNSUPPORTED, "P0-W Newton needs V = P1, W = P0");
      if (kind == EGFEM_INTERP_GRADPOW_P0 && !(p > 1.0))
        return fail(EGFEM_ERR_INVALID_ARGUMENT, "GRADPOW_P0 needs p > 1");
      if (check_ptrs && (st = check_dev_ptr(t, chain, "chain", true))) return st;
      *code = 3;
      return EGFEM_OK;
    case EGFEM_INTERP_RECIPROCAL:
      if (t->w_is_v) {
        if (!t->newton_wv_ok)
          return fail(EGFEM_ERR_UNSUPPORTED, "T·₂u has entries outside the CSR pattern (from_coo tensor)");
        *code = 2;
        return EGFEM_OK;
      }
      if (!t->has_mesh || !t->w_p0 || t->vfam != EGFEM_P1)
        return fail(EGFEM_ERR_UNSUPPORTED, "RECIPROCAL Newton needs W = V, or V = P1 and W = P0");
      if (check_ptrs && (st = check_dev_ptr(t, chain, "chain", true))) return st;
      *code = 3;
      return EGFEM_OK;
    case EGFEM_INTERP_P1_TO_P2_SQUARE:
      return fail(EGFEM_ERR_UNSUPPORTED, "NEWTON with P1_TO_P2_SQUARE is not implemented on the GPU");
    default:
      return fail(EGFEM_ERR_INVALID_ARGUMENT, "bad interp kind");
  }
}

egfem_status egfem_kernel_name(const egfem_tensor* t, int32_t entry, egfem_jac_mode mode, egfem_interp_kind kind,
                               double p, char* buf, size_t len) {
  if (!t || !buf || len == 0) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor or buffer is NULL");
  int code = 0;
  egfem_status st;
  if (entry == 1 || entry == 2)
    if ((st = jac_mode_code(t, mode, kind, p, nullptr, nullptr, &code, false))) return st;
  if (entry == 4 && (st = jac_mode_code(t, EGFEM_JAC_NEWTON, kind, p, nullptr, nullptr, &code, false))) return st;
  if (entry < 0 || entry > 5) return fail(EGFEM_ERR_INVALID_ARGUMENT, "entry must be 0..5");
  std::string name;
  if (entry == 5) {  // egfem_interp with kind
    const bool grad = kind == EGFEM_INTERP_GRADPOW_P0 || kind == EGFEM_INTERP_MINSURF_P0;
    if (grad && geo_interp_ok(t))
      name = "k_interp_gradpow_geo (" + std::to_string(t->n_geo) + " geometry classes, egfem_kernels.cu)";
    else if (grad)
      name = "k_interp_gradpow (egfem_kernels.cu)";
    else
      name = "k_interp_* (egfem_kernels.cu)";
  } else if (entry == 4)  // egfem_step (a 32-byte aligned chain assumed)
    name = step_path_ok(t, kind, nullptr) ? "k_step (single-pass interp + apply + Newton Jacobian, egfem_cells.cu)"
                                          : "k_interp_* + " + dispatch_name(t, 2, code);
  else
    name = dispatch_name(t, entry, code);
  std::snprintf(buf, len, "%s", name.c_str());
  return EGFEM_OK;
}

egfem_status egfem_group_compile(const int32_t* key, int32_t key_len, int32_t pairs_per_lane, int32_t f64) {
  if (!key || key_len < 2 || pairs_per_lane < 1 || pairs_per_lane > 4)
    return fail(EGFEM_ERR_INVALID_ARGUMENT, "group pattern key missing or pairs_per_lane out of [1, 4]");
  std::string log;
  egfem_status st = group_compile_key(key, key_len, pairs_per_lane, f64, &log);
  if (st == EGFEM_ERR_INVALID_ARGUMENT) return fail(st, "malformed group pattern key");
  return st;
}

// w may be NULL in a Newton call of a packed kind (GRADPOW_P0, MINSURF_P0 with chain) that the
// cell-major kernels serve: they read w_K from the packed record; any other call needs w.
static egfem_status check_w_newton(const egfem_tensor* t, int code, egfem_interp_kind kind, const void* w,
                                   const void* chain) {
  if (w) return check_dev_ptr(t, w, "w", true);
  if (code == 3 && chain && packed_chain_kind(kind) && cells_path_ok(t, code)) return EGFEM_OK;
  return fail(EGFEM_ERR_INVALID_ARGUMENT, "w is NULL (allowed only for a packed-kind Newton call on the cell-major path)");
}

egfem_status egfem_jacobian(const egfem_tensor* t, egfem_jac_mode mode, egfem_interp_kind kind, double p,
                            const void* u, const void* w, const void* chain, void* csr_vals, egfem_stream_t stream) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  egfem_status st;
  if ((st = check_dev_ptr(t, csr_vals, "csr_vals", true))) return st;
  int code = 0;
  if ((st = jac_mode_code(t, mode, kind, p, u, chain, &code))) return st;
  if ((st = check_w_newton(t, code, kind, w, chain))) return st;
  NvtxRange nv("egfem_jacobian");
  DeviceGuard g(t->device);
  return launch_tile(t, false, code, kind, p, u, w, chain, nullptr, csr_vals, (cudaStream_t)stream);
}

egfem_status egfem_apply_jacobian(const egfem_tensor* t, egfem_jac_mode mode, egfem_interp_kind kind, double p,
                                  const void* u, const void* w, const void* chain, void* r, void* csr_vals,
                                  egfem_stream_t stream) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  egfem_status st;
  if ((st = check_dev_ptr(t, u, "u", true)) || (st = check_dev_ptr(t, r, "r", true)) ||
      (st = check_dev_ptr(t, csr_vals, "csr_vals", true)))
    return st;
  int code = 0;
  if ((st = jac_mode_code(t, mode, kind, p, u, chain, &code))) return st;
  if ((st = check_w_newton(t, code, kind, w, chain))) return st;
  NvtxRange nv("egfem_apply_jacobian");
  DeviceGuard g(t->device);
  return launch_tile(t, true, code, kind, p, u, w, chain, r, csr_vals, (cudaStream_t)stream);
}

egfem_status egfem_step(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u, void* w, void* chain,
                        void* r, void* csr_vals, egfem_stream_t stream) {
  egfem_status st = interp_check(t, kind, p, u, w, chain);
  if (st) return st;
  if ((st = check_dev_ptr(t, r, "r", true)) || (st = check_dev_ptr(t, csr_vals, "csr_vals", true))) return st;
  int code = 0;
  if ((st = jac_mode_code(t, EGFEM_JAC_NEWTON, kind, p, u, chain, &code))) return st;
  if ((st = check_w_newton(t, code, kind, w, chain))) return st;
  NvtxRange nv("egfem_step");
  DeviceGuard g(t->device);
  const cudaStream_t s = (cudaStream_t)stream;
  st = launch_step(t, kind, p, u, w, chain, r, csr_vals, s);
  if (st != EGFEM_ERR_UNSUPPORTED) return st;
  // the tensor, kind or chain alignment does not fit the single-pass kernel: the two launches
  if ((st = launch_interp(t, kind, p, u, w, chain, 0, interp_items(t, kind), s))) return st;
  return launch_tile(t, true, code, kind, p, u, w, chain, r, csr_vals, s);
}

egfem_status egfem_apply_jacobian_rows(const egfem_tensor* t, egfem_jac_mode mode, egfem_interp_kind kind, double p,
                                       const void* u, const void* w, const void* chain, void* r, void* csr_vals,
                                       int64_t row_lo, int64_t row_hi, egfem_stream_t stream) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  egfem_status st;
  if ((st = check_dev_ptr(t, u, "u", true)) || (st = check_dev_ptr(t, r, "r", true)) ||
      (st = check_dev_ptr(t, csr_vals, "csr_vals", true)))
    return st;
  if (row_lo < 0 || row_hi < row_lo || row_hi > t->n_u)
    return fail(EGFEM_ERR_INVALID_ARGUMENT, "row range outside [0, n_u]");
  int code = 0;
  if ((st = jac_mode_code(t, mode, kind, p, u, chain, &code))) return st;
  if ((st = check_w_newton(t, code, kind, w, chain))) return st;
  NvtxRange nv("egfem_apply_jacobian_rows");
  DeviceGuard g(t->device);
  return launch_tile_rows(t, row_lo, row_hi, true, code, kind, p, u, w, chain, r, csr_vals, (cudaStream_t)stream);
}

egfem_status egfem_interior(const egfem_tensor* t, int64_t* row_lo, int64_t* row_hi, int64_t* w_lo, int64_t* w_hi) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  const bool all = t->int_row_lo < 0;  // global tensor: no halo
  const int64_t items = t->w_is_v ? t->n_f : t->n_cells;
  if (row_lo) *row_lo = all ? 0 : t->int_row_lo;
  if (row_hi) *row_hi = all ? t->n_u : t->int_row_hi;
  if (w_lo) *w_lo = all ? 0 : t->int_w_lo;
  if (w_hi) *w_hi = all ? items : t->int_w_hi;
  return EGFEM_OK;
}

egfem_status egfem_interior_rows(int64_t n_rows, const int64_t* row_ptr, const int32_t* col, int64_t own_lo,
                                 int64_t own_hi, int64_t* lo, int64_t* hi) {
  if (n_rows < 0 || !row_ptr || (!col && n_rows > 0 && row_ptr[n_rows] > 0) || !lo || !hi)
    return fail(EGFEM_ERR_INVALID_ARGUMENT, "bad arguments");
  int64_t best_lo = 0, best_hi = 0, run = -1;
  for (int64_t i = 0; i <= n_rows; ++i) {
    bool ok = i < n_rows;
    if (ok)
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
        if (col[e] < own_lo || col[e] >= own_hi) {
          ok = false;
          break;
        }
    if (ok && run < 0) run = i;
    if (!ok && run >= 0) {
      if (i - run > best_hi - best_lo) {
        best_lo = run;
        best_hi = i;
      }
      run = -1;
    }
  }
  *lo = best_lo;
  *hi = best_hi;
  return EGFEM_OK;
}

egfem_status egfem_bilinear_build(const egfem_tensor* t, void* b_vals, egfem_stream_t stream) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  egfem_status st;
  if ((st = check_dev_ptr(t, b_vals, "b_vals", true))) return st;
  if (!t->w_is_v) return fail(EGFEM_ERR_DIMENSION_MISMATCH, "bilinear form needs W = V numbering");
  if (!t->newton_wv_ok) return fail(EGFEM_ERR_UNSUPPORTED, "T·₂1 has entries outside the CSR pattern");
  if (t->int_row_lo >= 0)  // a local tensor of a partition: its columns are window indices
    return fail(EGFEM_ERR_UNSUPPORTED, "bilinear form of a partitioned tensor: build it on the global tensor");
  if (t->has_mesh && (t->form == EGFEM_FORM_CONV_J || t->form == EGFEM_FORM_PLAP))
    return fail(EGFEM_ERR_UNSUPPORTED, "the u-slot of this form is differentiated: T·₂1 = 0 (Σ_j ∇φ_j = 0)");
  NvtxRange nv("egfem_bilinear_build");
  DeviceGuard g(t->device);
  return launch_bilinear_build(t, b_vals, (cudaStream_t)stream);
}

egfem_status egfem_csr_spmv(const egfem_tensor* t, const void* vals, const void* x, void* y, egfem_stream_t stream) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  egfem_status st;
  if ((st = check_dev_ptr(t, vals, "vals", true)) || (st = check_dev_ptr(t, x, "x", true)) ||
      (st = check_dev_ptr(t, y, "y", true)))
    return st;
  if (x == y) return fail(EGFEM_ERR_INVALID_ARGUMENT, "x and y must not alias");
  NvtxRange nv("egfem_csr_spmv");
  DeviceGuard g(t->device);
  return launch_spmv(t, vals, x, y, (cudaStream_t)stream);
}

egfem_status egfem_bilinear_jacobian(const egfem_tensor* t, const void* b_vals, egfem_interp_kind kind, double p,
                                     const void* u, void* csr_vals, egfem_stream_t stream) {
  if (!t) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  egfem_status st;
  if ((st = check_dev_ptr(t, b_vals, "b_vals", true)) || (st = check_dev_ptr(t, u, "u", true)) ||
      (st = check_dev_ptr(t, csr_vals, "csr_vals", true)))
    return st;
  if (!t->w_is_v) return fail(EGFEM_ERR_DIMENSION_MISMATCH, "bilinear Jacobian needs W = V numbering");
  int mode = -1;
  if (kind == EGFEM_INTERP_IDENTITY) mode = 0;
  if (kind == EGFEM_INTERP_SQUARE) mode = 1;
  if (kind == EGFEM_INTERP_RECIPROCAL) mode = 2;
  if (mode < 0) return fail(EGFEM_ERR_UNSUPPORTED, "bilinear Jacobian: IDENTITY, SQUARE or RECIPROCAL");
  NvtxRange nv("egfem_bilinear_jacobian");
  DeviceGuard g(t->device);
  return launch_scale_cols(t, b_vals, mode, p, u, csr_vals, (cudaStream_t)stream);
}

egfem_status egfem_halo_pack(const egfem_tensor* local, const int32_t* d_idx, int64_t n, const void* u_local,
                             void* send_buf, egfem_stream_t stream) {
  if (!local) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  if (n < 0) return fail(EGFEM_ERR_INVALID_ARGUMENT, "n < 0");
  if (n == 0) return EGFEM_OK;
  egfem_status st;
  if ((st = check_dev_ptr(local, d_idx, "idx", true)) || (st = check_dev_ptr(local, u_local, "u_local", true)) ||
      (st = check_dev_ptr(local, send_buf, "send_buf", true)))
    return st;
  NvtxRange nv("egfem_halo_pack");
  DeviceGuard g(local->device);
  return launch_halo(local, d_idx, n, u_local, send_buf, true, (cudaStream_t)stream);
}

egfem_status egfem_halo_unpack(const egfem_tensor* local, const int32_t* d_idx, int64_t n, const void* recv_buf,
                               void* u_local, egfem_stream_t stream) {
  if (!local) return fail(EGFEM_ERR_INVALID_ARGUMENT, "tensor is NULL");
  if (n < 0) return fail(EGFEM_ERR_INVALID_ARGUMENT, "n < 0");
  if (n == 0) return EGFEM_OK;
  egfem_status st;
  if ((st = check_dev_ptr(local, d_idx, "idx", true)) || (st = check_dev_ptr(local, recv_buf, "recv_buf", true)) ||
      (st = check_dev_ptr(local, u_local, "u_local", true)))
    return st;
  NvtxRange nv("egfem_halo_unpack");
  DeviceGuard g(local->device);
  return launch_halo(local, d_idx, n, recv_buf, u_local, false, (cudaStream_t)stream);
}

// ------------------------------------------------------------------ partition
egfem_status egfem_partition_rows(int64_t n_rows, const int64_t* prefix, int32_t nranks, int64_t* bounds) {
  if (n_rows < 0 || !prefix || !bounds || nranks < 1) return fail(EGFEM_ERR_INVALID_ARGUMENT, "bad arguments");
  // Rank r owns rows [bounds[r], bounds[r+1]): the first row whose prefix reaches
  // r·nnz/nranks (ceil) starts rank r.  Deterministic and monotone.
  const int64_t total = prefix[n_rows];
  bounds[0] = 0;
  for (int32_t r = 1; r < nranks; ++r) {
    const int64_t target = (total * r + nranks - 1) / nranks;
    const int64_t* p = std::lower_bound(prefix, prefix + n_rows + 1, target);
    int64_t row = (int64_t)(p - prefix);
    row = std::min<int64_t>(std::max<int64_t>(row, bounds[r - 1]), n_rows);
    bounds[r] = row;
  }
  bounds[nranks] = n_rows;
  return EGFEM_OK;
}

egfem_status egfem_partition(const egfem_tensor* G, int32_t nranks, int32_t rank, int device, egfem_tensor** out,
                             int64_t* row_begin, int64_t* row_end, int64_t* col_begin, int64_t* col_end,
                             int64_t* w_begin, int64_t* w_end) {
  if (!G || !out) return fail(EGFEM_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(EGFEM_ERR_INVALID_ARGUMENT, "bad rank / nranks");
  if (device != G->device) return fail(EGFEM_ERR_UNSUPPORTED, "partition onto another device");
  if (G->has_mesh && !G->w_p0 && !G->w_is_v)
    return fail(EGFEM_ERR_UNSUPPORTED, "row partition needs W = V or W = P0");
  if (G->wfam == EGFEM_QUAD) return fail(EGFEM_ERR_UNSUPPORTED, "row partition of QUAD W is not implemented");
  NvtxRange nv("egfem_partition");
  DeviceGuard g(G->device);
  // host copies of the integer structure (offline)
  std::vector<int64_t> row_fib(G->n_u + 1);
  std::vector<uint32_t> fib_nz(G->n_fib + 1);
  EGFEM_CUDA_TRY(cudaMemcpy(row_fib.data(), G->row_fib, 8 * (G->n_u + 1), cudaMemcpyDeviceToHost));
  EGFEM_CUDA_TRY(cudaMemcpy(fib_nz.data(), G->fib_nz, 4 * (G->n_fib + 1), cudaMemcpyDeviceToHost));
  std::vector<int64_t> prefix(G->n_u + 1);
  for (int64_t i = 0; i <= G->n_u; ++i) prefix[i] = fib_nz[row_fib[i]];
  std::vector<int64_t> bounds(nranks + 1);
  egfem_partition_rows(G->n_u, prefix.data(), nranks, bounds.data());
  const int64_t rb = bounds[rank], re = bounds[rank + 1];
  const int64_t f0 = row_fib[rb], f1 = row_fib[re];
  const int64_t e0 = fib_nz[f0], e1 = fib_nz[f1];
  const int64_t nf = f1 - f0, ne = e1 - e0, nr = re - rb;
  std::vector<int32_t> fj(nf);
  std::vector<uint32_t> nk(ne);
  if (nf) EGFEM_CUDA_TRY(cudaMemcpy(fj.data(), G->fib_j + f0, 4 * nf, cudaMemcpyDeviceToHost));
  if (ne) EGFEM_CUDA_TRY(cudaMemcpy(nk.data(), G->nz_k + e0, 4 * ne, cudaMemcpyDeviceToHost));
  int64_t cb = rb, ce = re;  // column window includes the owned rows
  for (int32_t j : fj) {
    cb = std::min<int64_t>(cb, j);
    ce = std::max<int64_t>(ce, (int64_t)j + 1);
  }
  const bool p0 = G->has_mesh && G->w_p0;
  std::vector<int32_t> wlist;  // P0: referenced cells, ascending
  if (p0) {
    wlist.reserve(ne / 4 + 1);
    for (uint32_t x : nk) wlist.push_back((int32_t)(x & kKMask));
    std::sort(wlist.begin(), wlist.end());
    wlist.erase(std::unique(wlist.begin(), wlist.end()), wlist.end());
  } else {
    for (uint32_t x : nk) {  // W = V: k lies in the column window
      const int64_t k = x & kKMaskAny;
      cb = std::min<int64_t>(cb, k);
      ce = std::max<int64_t>(ce, k + 1);
    }
  }
  // local arrays
  egfem_tensor* t = new egfem_tensor();
  t->device = device;
  t->dtype = G->dtype;
  t->form = G->form;
  t->dim = G->dim;
  t->vfam = G->vfam;
  t->wfam = G->wfam;
  t->nV = G->nV;
  t->nW = G->nW;
  t->n_u = nr;  // local rows
  t->nnz = ne;
  t->n_fib = nf;
  t->row_begin = rb;
  t->col_begin = cb;
  t->w_is_v = G->w_is_v;
  t->w_p0 = G->w_p0;
  t->newton_wv_ok = G->newton_wv_ok;
  const int64_t n_local = ce - cb;
  auto bail = [&](egfem_status s) {
    free_tensor(t);
    delete t;
    return s;
  };
  std::vector<int64_t> lrf(nr + 1);
  for (int64_t i = 0; i <= nr; ++i) lrf[i] = row_fib[rb + i] - f0;
  std::vector<uint32_t> lfn(nf + 1);
  for (int64_t f = 0; f <= nf; ++f) lfn[f] = (uint32_t)(fib_nz[f0 + f] - e0);
  for (auto& j : fj) j = (int32_t)(j - cb);
  if (p0) {
    for (auto& x : nk) {
      const int32_t K = (int32_t)(x & kKMask);
      const int32_t lk = (int32_t)(std::lower_bound(wlist.begin(), wlist.end(), K) - wlist.begin());
      x = (uint32_t)lk | (x & ~kKMask);
    }
    t->n_f = (int64_t)wlist.size();
  } else {
    for (auto& x : nk) x = (uint32_t)((int64_t)(x & kKMaskAny) - cb) | (x & kHead);
    t->n_f = n_local;
  }
  // NOTE: the local column space has n_local entries; rows are a prefix-free subset.
  const size_t vs = t->dtype == EGFEM_F64 ? 8 : 4;
  std::vector<int64_t> lrn(nr + 1);
  for (int64_t i = 0; i <= nr; ++i) lrn[i] = (int64_t)lfn[lrf[i]];
  if (dmalloc_padded((void**)&t->row_nz, 8 * (nr + 1)) ||
      cudaMemcpy(t->row_nz, lrn.data(), 8 * (nr + 1), cudaMemcpyHostToDevice))
    return bail(fail(EGFEM_ERR_OUT_OF_MEMORY, "row_nz upload failed"));
  if (dmalloc_padded((void**)&t->row_fib, 8 * (nr + 1)) || dmalloc_padded((void**)&t->fib_j, 4 * nf) ||
      dmalloc_padded((void**)&t->fib_nz, 4 * (nf + 1)) || dmalloc_padded((void**)&t->nz_k, 4 * ne) ||
      dmalloc_padded(&t->nz_val, vs * ne) || (p0 && dmalloc_padded((void**)&t->nz_aux, ne)))
    return bail(fail(EGFEM_ERR_OUT_OF_MEMORY, "cudaMalloc failed"));
  if (p0 && ne && cudaMemcpy(t->nz_aux, G->nz_aux + e0, ne, cudaMemcpyDeviceToDevice))
    return bail(fail(EGFEM_ERR_CUDA, "cudaMemcpy failed"));
  if (cudaMemcpy(t->row_fib, lrf.data(), 8 * (nr + 1), cudaMemcpyHostToDevice) ||
      (nf && cudaMemcpy(t->fib_j, fj.data(), 4 * nf, cudaMemcpyHostToDevice)) ||
      cudaMemcpy(t->fib_nz, lfn.data(), 4 * (nf + 1), cudaMemcpyHostToDevice) ||
      (ne && cudaMemcpy(t->nz_k, nk.data(), 4 * ne, cudaMemcpyHostToDevice)) ||
      (ne && cudaMemcpy(t->nz_val, (const char*)G->nz_val + vs * e0, vs * ne, cudaMemcpyDeviceToDevice)))
    return bail(fail(EGFEM_ERR_CUDA, "cudaMemcpy failed"));
  // local mesh data for GRADPOW interp: referenced cells with local vertex ids
  if (p0) {
    t->has_mesh = true;
    const int d1 = G->dim + 1;
    const int64_t ncl = (int64_t)wlist.size();
    t->n_cells = ncl;
    t->n_vertices = n_local;
    std::vector<int32_t> gcells(G->n_cells * d1), gv(G->n_cells * G->nV);
    EGFEM_CUDA_TRY(cudaMemcpy(gcells.data(), G->cells, 4 * gcells.size(), cudaMemcpyDeviceToHost));
    EGFEM_CUDA_TRY(cudaMemcpy(gv.data(), G->vdofs, 4 * gv.size(), cudaMemcpyDeviceToHost));
    std::vector<int32_t> gwcell(G->n_f);
    EGFEM_CUDA_TRY(cudaMemcpy(gwcell.data(), G->wcell, 4 * G->n_f, cudaMemcpyDeviceToHost));
    std::vector<int32_t> lc(ncl * d1), lv(ncl * G->nV), lw(ncl);
    for (int64_t c = 0; c < ncl; ++c) {
      const int64_t gc = gwcell[wlist[c]];
      for (int a = 0; a < d1; ++a) {
        const int64_t v = gcells[gc * d1 + a] - cb;
        if (v < 0 || v >= n_local) return bail(fail(EGFEM_ERR_UNSUPPORTED, "cell vertex outside the halo window"));
        lc[c * d1 + a] = (int32_t)v;
      }
      for (int a = 0; a < G->nV; ++a) lv[c * G->nV + a] = gv[gc * G->nV + a] - (int32_t)cb;
      lw[c] = (int32_t)c;
    }
    // P1 geometry: vertex ids are V dofs, coordinates of the window [cb, ce)
    if (cudaMalloc(&t->coords, 8 * std::max<int64_t>(n_local * G->dim, 1)) ||
        cudaMalloc(&t->cells, 4 * std::max<int64_t>(ncl * d1, 1)) ||
        cudaMalloc(&t->vdofs, 4 * std::max<int64_t>(ncl * G->nV, 1)) ||
        cudaMalloc(&t->wdofs, 4 * std::max<int64_t>(ncl, 1)) || cudaMalloc(&t->wcell, 4 * std::max<int64_t>(ncl, 1)))
      return bail(fail(EGFEM_ERR_OUT_OF_MEMORY, "cudaMalloc failed"));
    t->vdofs_is_cells = G->vdofs_is_cells;
    t->wdofs_is_iota = true;
    t->nwc = 1;
    if (cudaMalloc(&t->wpts, sizeof(double) * d1) ||
        cudaMemcpy(t->wpts, G->wpts, sizeof(double) * d1, cudaMemcpyDeviceToDevice))
      return bail(fail(EGFEM_ERR_CUDA, "wpts copy failed"));
    if (G->dim == 3 && (cudaMalloc(&t->coords4, 32 * std::max<int64_t>(n_local, 1)) ||
                        cudaMemcpy(t->coords4, G->coords4 + cb * 4, 32 * n_local, cudaMemcpyDeviceToDevice)))
      return bail(fail(EGFEM_ERR_CUDA, "coords4 copy failed"));
    const int cfs = G->dim == 3 ? 4 : 2;  // floats per vertex of the exact float copy
    if (G->coordsf && (cudaMalloc(&t->coordsf, 4 * cfs * std::max<int64_t>(n_local, 1)) ||
                       cudaMemcpy(t->coordsf, G->coordsf + cb * cfs, 4 * cfs * n_local, cudaMemcpyDeviceToDevice)))
      return bail(fail(EGFEM_ERR_CUDA, "coordsf copy failed"));
    if (cudaMemcpy(t->coords, G->coords + cb * G->dim, 8 * n_local * G->dim, cudaMemcpyDeviceToDevice) ||
        (ncl && cudaMemcpy(t->cells, lc.data(), 4 * lc.size(), cudaMemcpyHostToDevice)) ||
        (ncl && cudaMemcpy(t->vdofs, lv.data(), 4 * lv.size(), cudaMemcpyHostToDevice)) ||
        (ncl && cudaMemcpy(t->wdofs, lw.data(), 4 * lw.size(), cudaMemcpyHostToDevice)) ||
        (ncl && cudaMemcpy(t->wcell, lw.data(), 4 * lw.size(), cudaMemcpyHostToDevice)))
      return bail(fail(EGFEM_ERR_CUDA, "cudaMemcpy failed"));
  }
  // interior / boundary split (egfem_interior): rows reading only owned u, and the interp
  // items covering their w that read only owned u
  {
    const int64_t olo = rb - cb, ohi = re - cb;
    std::vector<int32_t> kcol;  // per nonzero: the u index its w depends on (W = V: k), for the run test
    int64_t ia = 0, ib = 0;
    egfem_interior_rows(nr, lrf.data(), fj.data(), olo, ohi, &ia, &ib);
    if (!p0) {
      // W = V: the k of every nonzero of a run row must be owned too; shrink the run to its
      // longest sub-run with that property
      std::vector<int64_t> rp(ib - ia + 1);
      for (int64_t i = ia; i <= ib; ++i) rp[i - ia] = lfn[lrf[i]] - lfn[lrf[ia]];
      kcol.resize(rp.back());
      for (int64_t e = 0; e < (int64_t)kcol.size(); ++e) kcol[e] = (int32_t)(nk[lfn[lrf[ia]] + e] & kKMaskAny);
      int64_t a = 0, b = 0;
      egfem_interior_rows(ib - ia, rp.data(), kcol.data(), olo, ohi, &a, &b);
      ib = ia + b;
      ia = ia + a;
      t->int_w_lo = ia < ib ? olo : 0;
      t->int_w_hi = ia < ib ? ohi : 0;
    } else if (ia < ib) {
      // P0: the cells of rows [ia, ib) (local cell ids ascend with the global ones) must read
      // owned vertices only, and so must every cell between them (one contiguous item range)
      int64_t ca = INT64_MAX, cz = -1;
      for (int64_t e = lfn[lrf[ia]]; e < (int64_t)lfn[lrf[ib]]; ++e) {
        const int64_t c = nk[e] & kKMask;
        ca = std::min(ca, c);
        cz = std::max(cz, c);
      }
      bool ok = cz >= ca;
      if (ok) {
        const int d1 = G->dim + 1;
        std::vector<int32_t> hc(d1 * (cz + 1 - ca));
        ok = cudaMemcpy(hc.data(), t->cells + ca * d1, 4 * hc.size(), cudaMemcpyDeviceToHost) == cudaSuccess;
        for (size_t q = 0; ok && q < hc.size(); ++q) ok = hc[q] >= olo && hc[q] < ohi;
      }
      t->int_w_lo = ok ? ca : 0;
      t->int_w_hi = ok ? cz + 1 : 0;
      if (!ok) ia = ib = 0;
    } else {
      t->int_w_lo = t->int_w_hi = 0;
    }
    t->int_row_lo = ia;
    t->int_row_hi = ib;
  }
  // tiles of the local rows
  {
    egfem_status st = make_tiles(t, lrf, lfn);
    if (st) return bail(st);
    if ((st = make_wv_aux(t))) return bail(st);
    if ((st = make_p0_cells(t))) return bail(st);
    if ((st = make_dense_blocks(t, lrf))) return bail(st);
    // compiled row groups of the local rows (their columns are window indices: make_groups maps a
    // column to its local row by the window offset) — the row-partitioned batched action
    if ((st = make_groups(t, lrf))) return bail(st);
  }
  if (row_begin) *row_begin = rb;
  if (row_end) *row_end = re;
  if (col_begin) *col_begin = cb;
  if (col_end) *col_end = ce;
  if (w_begin) *w_begin = p0 ? (wlist.empty() ? 0 : wlist.front()) : cb;
  if (w_end) *w_end = p0 ? (wlist.empty() ? 0 : wlist.back() + 1) : ce;
  *out = t;
  return EGFEM_OK;
}

}  // extern "C"

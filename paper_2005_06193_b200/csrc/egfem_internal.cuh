// Internal definitions of libegfem.so (B200 / sm_100a).  Not part of the ABI.
//
// Device layout of a tensor: a fiber-compressed (CSF) T,
//   rows i -> fibers (i, j) -> nonzeros (k, value),
// whose fibers coincide one-to-one with the CSR slots of the Jacobian pattern:
//   row_fib[i] .. row_fib[i+1]   fibers of row i      (== csr_row_ptr)
//   fib_j[f]                     column j of fiber f   (== csr_col)
//   fib_nz[f] .. fib_nz[f+1]     nonzeros of fiber f   (uint32 offsets)
//   nz_k[e]                      k; bit 31 flags the first nonzero of a fiber; for
//                                W = P0 bits 28-29 hold loc_j (local index of j in cell k)
//   row_nz[i]                    first nonzero of row i (== canonical t_row_ptr)
//   nz_val[e]                    T_ijk in the handle dtype
// Rows are grouped into tiles (tile_row) of at most kTileNnz nonzeros, kTileFib
// fibers and kTileRows rows; one CTA processes one tile entirely in shared memory.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <array>
#include <mutex>
#include <string>
#include <vector>

#include "egfem.h"

namespace egfem {
struct GroupPlan;  // egfem_group.cu: compiled row-group kernels of the batched action
struct StepPlan;   // egfem_cells.cu: work order of the single-pass Newton step kernel

constexpr int kTileNnz = 1024;   // max nonzeros per tile
constexpr int kTileFib = 512;    // max fibers per tile
constexpr int kTileRows = 256;   // max rows per tile
constexpr int kThreads = 256;    // CTA size of the tile kernels
constexpr int kKShift = 28;      // loc_j packing in nz_k for P0 W (bits 28-29)
constexpr uint32_t kKMask = (1u << kKShift) - 1u;   // k of a P0-W tensor
constexpr uint32_t kKMaskAny = 0x7FFFFFFFu;          // k of any other tensor
constexpr uint32_t kHead = 0x80000000u;              // bit 31: first nonzero of a fiber
constexpr int kMaxQuad = 16;
constexpr int kMaxGeoClasses = 32;  // geometry classes of the 3D interp (egfem_tensor::gcls)
constexpr int kRowsMaxNnz = 512;   // rows up to this length take the row-group path (k_seg)
// cell-major copy: ck_b packs the fiber index within the row (6 bits) and the canonical position
// within the row (10 bits)
constexpr int kCellsMaxNnz = 1024;
constexpr uint32_t kCkFibMask = 63u;
constexpr int kCkPosShift = 6;
constexpr int kWVMaxNnz = 256;     // W = V Newton transpose data: position in a row fits 8 bits

void set_error(const std::string& msg);
void count_launch(int n = 1);
void count_launch_kernel(const char* name);

}  // namespace egfem

struct egfem_tensor {
  int device = 0;
  egfem_dtype dtype = EGFEM_F64;
  bool has_mesh = false;
  int dim = 0;
  int64_t n_u = 0, n_f = 0, n_cells = 0, n_vertices = 0;
  egfem_family vfam = EGFEM_P1, wfam = EGFEM_P1;
  int nV = 0, nW = 0;
  egfem_form form = EGFEM_FORM_CONV_J;
  int64_t nnz = 0, n_fib = 0;
  bool w_is_v = false;   // W numbering identical to V numbering (IDENTITY/SQUARE allowed)
  bool w_p0 = false;     // cell-wise W (P0 or QUAD): every W DOF lies in one cell (loc packed into nz_k)
  int nwc = 1;           // W DOFs per cell of a cell-wise W (P0: 1, QUAD: N_q)
  double* wpts = nullptr;  // cell-wise W: barycentric coordinates of a cell's W DOFs, nwc*(dim+1) (device)
  bool newton_wv_ok = false;  // every (i, k) of T is an (i, j) fiber (T·₂u fits the CSR pattern)
  int max_row_nnz = 0, max_row_fib = 0;
  uint32_t kmask() const { return (has_mesh && w_p0) ? egfem::kKMask : egfem::kKMaskAny; }

  // CSF tensor (device)
  int64_t* row_fib = nullptr;   // n_u+1
  int64_t* row_nz = nullptr;    // n_u+1 (first nonzero of each row)
  int32_t* fib_j = nullptr;     // n_fib
  uint32_t* fib_nz = nullptr;   // n_fib+1
  uint32_t* nz_k = nullptr;     // nnz
  void* nz_val = nullptr;       // nnz, dtype
  uint8_t* nz_aux = nullptr;    // nnz, P0 W only: position of k among the cells of row i
  uint8_t* nz_kpos = nullptr;   // nnz, W = V only: position of the nonzero in its row's (k, j) order
  uint8_t* fib_kr = nullptr;    // n_fib, W = V only: start of fiber (i, m)'s k = m run in that order
  // P0 W only: the same nonzeros in cell-major order (rows -> cells K ascending -> local vertex m)
  uint32_t* ck_k = nullptr;     // nnz/(d+1): K of each row cell
  void* ck_val = nullptr;       // nnz, dtype: T_{i v_m K}
  uint16_t* ck_b = nullptr;     // nnz: fiber index within the row | canonical position << 6
  // the same per-cell data packed into one 64-bit word per row cell when it fits (make_p0_cells):
  // bits [m·FW, m·FW + FB) fiber of nonzero m, [m·FW + FB, (m+1)·FW) its canonical position
  // (FW = FB + PB), bits [ck_ks, 64) K − ck_kb[row]; the kernel reads it straight into registers
  uint64_t* ck_m = nullptr;     // nnz/(d+1)
  uint32_t* ck_kb = nullptr;    // n_u: K of each row's first cell (cells ascend: the minimum)
  int ck_fb = 0, ck_pb = 0, ck_ks = 0;
  // W = V only (batched action): per row the dense |N|x|N| block over its CSR stencil N(i)
  int64_t* blk_off = nullptr;   // n_u+1: block offsets (row stride |N| rounded up to even)
  void* blk = nullptr;          // dtype: M_i[a][b] = T_{i, N_a, N_b}
  void* blk_sym = nullptr;      // dtype: (M_i + M_iᵀ)[a][b] (the IDENTITY Newton with u == w, k_dense1)
  int32_t* dense_rows = nullptr;  // n_u: rows grouped by stencil width |N(i)| (row order within a width)
  std::vector<std::array<int64_t, 4>> dense_classes;  // host: (width, first entry in dense_rows, count, first block value)
  egfem::GroupPlan* grp = nullptr;  // W = V batched action: row groups with compiled-in patterns (egfem_group.cu)
  egfem::StepPlan* step = nullptr;  // canonical P0 W: single-pass interp + Newton step (egfem_cells.cu)

  // tiles (device + host copy of the count)
  int32_t n_tiles = 0;
  int64_t* tile_row = nullptr;  // n_tiles+1 first row of each tile
  int64_t* tile_fib = nullptr;  // n_tiles+1 first fiber
  int64_t* tile_nz = nullptr;   // n_tiles+1 first nonzero

  // interpolation data (device): geometry in fp64 regardless of dtype
  double* coords = nullptr;     // n_vertices*dim
  double* coords4 = nullptr;    // 3D only: n_vertices*4 (x, y, z, 0) for 32-byte vector loads
  float* coordsf = nullptr;     // 2D/3D, when every coordinate is exactly a float: float2 (x, y) / float4 (x, y, z, 0) copy (lossless)
  bool vdofs_is_cells = false;  // V DOF table == mesh cell table (canonical P1)
  bool wdofs_is_iota = false;   // W DOF l of cell c is c·nW + l (canonical P0 / QUAD)
  int32_t* cells = nullptr;     // n_cells*(dim+1) mesh vertex ids (geometry)
  int32_t* vdofs = nullptr;     // n_cells*nV  V dof ids (u indices)
  int32_t* wdofs = nullptr;     // n_cells*nW  W dof ids
  int32_t* wcell = nullptr;     // n_f: cell owning P0 dof k (P0 W only)
  // geometry classes (3D, canonical P1 V / P0 W, at most kMaxGeoClasses): cells whose edge vectors
  // x_{a+1} − x_0 are bitwise equal share one entry (egfem_build.cu make_geo_classes)
  uint8_t* gcls = nullptr;      // n_cells: class of each cell
  double* gtab = nullptr;       // 10 x n_geo: cc[a][q] (v = 3a + q) and 1/det (v = 9) of each class
  int n_geo = 0;

  // partition bookkeeping (global handles: 0 / identity)
  int64_t row_begin = 0, col_begin = 0;
  // local tensors: rows / interp items that read only owned u (egfem_interior); -1 = all
  int64_t int_row_lo = -1, int_row_hi = -1, int_w_lo = -1, int_w_hi = -1;

  // caller pointers already validated on this handle (check_dev_ptr): a hit skips the driver's
  // cudaPointerGetAttributes, so a step's repeated calls on the same buffers cost no driver query
  mutable std::mutex ptr_mu;
  mutable uintptr_t ptr_ok[16] = {};
  mutable int ptr_ok_next = 0;
};

namespace egfem {

// builder / export (egfem_build.cu)
egfem_status build_from_triples(egfem_tensor* t, int64_t m, uint64_t* d_key_ij, uint32_t* d_k, double* d_val);
egfem_status upload_mesh(egfem_tensor* t, const egfem_mesh* mesh, const egfem_space* V, const egfem_space* W);
egfem_status make_geo_classes(egfem_tensor* t, const egfem_mesh* mesh);
// the interp of the gradient kinds reads geometry classes (handles with a class table)
inline bool geo_interp_ok(const egfem_tensor* t) {
  return t->dim == 3 && t->gcls && t->vdofs_is_cells && t->wdofs_is_iota && t->nwc == 1;
}
egfem_status emit_element_triples(egfem_tensor* t, egfem_form form, const egfem_quad* quad, int64_t* m_out,
                                  uint64_t** key, uint32_t** k, double** val);
egfem_status export_arrays(const egfem_tensor* t, int64_t* t_row_ptr, int32_t* t_j, int32_t* t_k, void* t_val,
                           int64_t* csr_row_ptr, int32_t* csr_col, int32_t* slot_ij, int32_t* slot_ik,
                           uint8_t* loc);
void free_tensor(egfem_tensor* t);
egfem_status make_tiles(egfem_tensor* t, const std::vector<int64_t>& row_fib_h, const std::vector<uint32_t>& fib_nz_h);
cudaError_t dmalloc_padded(void** p, size_t bytes);

// compute kernels (egfem_kernels.cu)
egfem_status launch_interp(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u, void* w,
                           void* chain, int64_t lo, int64_t hi, cudaStream_t s);
int64_t interp_items(const egfem_tensor* t, egfem_interp_kind kind);
egfem_status launch_tile_rows(const egfem_tensor* t, int64_t lo, int64_t hi, bool do_r, int jac,
                              egfem_interp_kind kind, double p, const void* u, const void* w, const void* chain,
                              void* r, void* csr_vals, cudaStream_t s);
egfem_status launch_tile(const egfem_tensor* t, bool do_r, int jac, egfem_interp_kind kind, double p, const void* u,
                         const void* w, const void* chain, void* r, void* csr_vals, cudaStream_t s);
egfem_status launch_rows(const egfem_tensor* t, bool do_r, int jac, egfem_interp_kind kind, double p, const void* u,
                         const void* w, const void* chain, void* r, void* csr_vals, cudaStream_t s);
bool rows_path_ok(const egfem_tensor* t, int jac);
egfem_status make_wv_aux(egfem_tensor* t);
bool cells_path_ok(const egfem_tensor* t, int jac);
const char* cells_variant(const egfem_tensor* t);
egfem_status launch_cells(const egfem_tensor* t, bool do_r, int jac, bool packed, const void* u, const void* w,
                          const void* chain, void* r, void* csr_vals, cudaStream_t s);
egfem_status make_p0_cells(egfem_tensor* t);
// single-pass Newton step (interp of the gradient kinds + fused apply / Newton Jacobian in one
// launch, egfem_cells.cu): the plan is built with the tensor when it applies; launch_step returns
// EGFEM_ERR_UNSUPPORTED (nothing launched) when the tensor, kind or pointers do not fit it
egfem_status make_step_plan(egfem_tensor* t);
void free_step_plan(StepPlan* sp);
bool step_path_ok(const egfem_tensor* t, egfem_interp_kind kind, const void* chain);
egfem_status launch_step(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u, void* w, void* chain,
                         void* r, void* csr_vals, cudaStream_t s);
bool dense_path_ok(const egfem_tensor* t);
bool dense1_path_ok(const egfem_tensor* t, int jac);
egfem_status launch_dense1(const egfem_tensor* t, int64_t lo, int64_t hi, bool do_r, int jac, egfem_interp_kind kind,
                           double p, const void* u, const void* w, void* r, void* csr_vals, cudaStream_t s);
egfem_status launch_dense(const egfem_tensor* t, int32_t batch, egfem_layout layout, const void* U, const void* W,
                          void* R, cudaStream_t s);
egfem_status make_dense_blocks(egfem_tensor* t, const std::vector<int64_t>& hrf);
egfem_status launch_dense_rows(const egfem_tensor* t, int32_t batch, const int32_t* rows,
                               const std::vector<std::array<int64_t, 3>>& classes, const void* U, const void* W,
                               void* R, cudaStream_t s);
// grouped batched action with compiled patterns (egfem_group.cu)
egfem_status make_groups(egfem_tensor* t, const std::vector<int64_t>& hrf);
void free_group_plan(GroupPlan* gp);
bool group_path_ok(const egfem_tensor* t, egfem_layout layout);
egfem_status launch_groups(const egfem_tensor* t, int32_t batch, const void* U, const void* W, void* R,
                           cudaStream_t s);
const char* group_plan_info(const egfem_tensor* t);
// the gradient kinds' Newton data is the packed chain record [w_k, ∂w/∂u_0 .. ∂w/∂u_{d−1}]
// (include/egfem.h egfem_interp); the other cell-wise kinds store D_u w in full
inline bool packed_chain_kind(egfem_interp_kind kind) {
  return kind == EGFEM_INTERP_GRADPOW_P0 || kind == EGFEM_INTERP_MINSURF_P0;
}
egfem_status group_compile_key(const int32_t* key, int32_t len, int P, int f64, std::string* log);
// the kernel family an entry point dispatches to (0 apply, 1 jacobian, 2 apply_jacobian,
// 3 apply_batched node-major; jac = the Jacobian mode code)
std::string dispatch_name(const egfem_tensor* t, int entry, int jac);
egfem_status launch_spmv(const egfem_tensor* t, const void* vals, const void* x, void* y, cudaStream_t s);
egfem_status launch_scale_cols(const egfem_tensor* t, const void* b, int mode, double p, const void* u, void* J,
                               cudaStream_t s);
egfem_status launch_bilinear_build(const egfem_tensor* t, void* b_vals, cudaStream_t s);
egfem_status launch_batched(const egfem_tensor* t, int32_t batch, egfem_layout layout, const void* U,
                            const void* W, void* R, cudaStream_t s);
egfem_status launch_halo(const egfem_tensor* t, const int32_t* idx, int64_t n, const void* src, void* dst,
                         bool pack, cudaStream_t s);

}  // namespace egfem

#define EGFEM_CUDA_TRY(expr)                                                                  \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess) {                                                                  \
      egfem::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                 \
      return _e == cudaErrorMemoryAllocation ? EGFEM_ERR_OUT_OF_MEMORY : EGFEM_ERR_CUDA;      \
    }                                                                                         \
  } while (0)

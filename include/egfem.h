/*
 * egfem.h — C ABI of libegfem.so, the B200 (sm_100a) hot path of the extended
 * group finite element method (EGFEM, Tolle & Marheineke, arXiv 2005.06193).
 *
 * The method replaces each nonlinear coefficient f(u, ∇u) by its interpolant on a
 * space W_h tailored to the nonlinearity (§3.1, eq. (egfem_coeffs)),
 * which turns the nonlinear residual into trilinear forms held as assembled sparse
 * third-order tensors T_ijk (eq. (egfem_terms)).  Each Picard or
 * Newton iteration then needs only
 *   (1) w = f(Π_u u, Π_∇u ·₂ u)                       egfem_interp
 *   (2) r_i = (T:(u⊗w))_i = Σ_jk T_ijk u_j w_k        egfem_apply
 *   (3) A = T·w, or J = T·w + (T·₂u)·D_u w             egfem_jacobian
 * on a tensor precomputed once                         egfem_tensor_build ("offline").
 *
 * Conventions for every function:
 *   - Every function returns egfem_status; none throws, aborts or exits.
 *   - Validation (null / misaligned pointers, wrong device, bad enum, size or index
 *     overflow) happens synchronously BEFORE any launch; on a validation error no
 *     output is written.  egfem_last_error() returns a thread-local detail string.
 *   - Mesh / space / quadrature arrays passed to egfem_tensor_build are HOST
 *     pointers, copied during the call; the caller may free them afterwards.
 *   - u, w, r, chain, csr_vals, U, W, R are caller-owned DEVICE pointers on the
 *     handle's device, of the handle's dtype, 16-byte aligned, contiguous.
 *     Lengths are implied by egfem_tensor_info (N_u, N_f, nnz_csr).
 *     Each handle remembers the last 16 device pointers that passed the device check
 *     (cudaPointerGetAttributes); a remembered pointer is not queried again, so a
 *     buffer freed with cudaFree after use on a handle must not be passed to it again.
 *   - Compute calls are asynchronous on the given cudaStream_t (0 = legacy default).
 *     Kernel faults surface at the next call or at the caller's stream sync.
 *   - The handle is immutable after build (its only lazily created state — the compiled
 *     batched kernels and their side streams — is created under a lock on first use);
 *     interp/apply/jacobian are pure functions of their inputs and may run concurrently
 *     on different streams.
 *   - No floating-point atomics: results are bitwise reproducible run to run.
 *   - csr_vals is fully overwritten, never accumulated into.
 *   - Tracing: every compute call opens an NVTX range named after the function for the
 *     duration of the host call (a no-op without an attached profiler).
 */
#ifndef EGFEM_H
#define EGFEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* egfem_stream_t; /* == cudaStream_t */

typedef enum {
  EGFEM_OK = 0,
  EGFEM_ERR_INVALID_ARGUMENT = 1,
  EGFEM_ERR_DIMENSION_MISMATCH = 2,
  EGFEM_ERR_UNSUPPORTED = 3,
  EGFEM_ERR_INDEX_OVERFLOW = 4,
  EGFEM_ERR_OUT_OF_MEMORY = 5,
  EGFEM_ERR_CUDA = 6,
  EGFEM_ERR_NCCL = 7
} egfem_status;

typedef enum { EGFEM_F64 = 0, EGFEM_F32 = 1 } egfem_dtype;

/* Families.  P0/P1/P2: Lagrange (P0 for gradient nonlinearities
 * L584).  QUAD: the quadrature-embedded space I_k of Case 3 (L117–139, eq.
 * (quadrature_basis)), W only: its DOFs are the N_q points x_ℓ^K of the rule used for
 * the assembly in every cell (N_f = N_q·N_el, L139), basis η_ℓ^K = w_ℓ^K δ_{x_ℓ^K}, so
 * T_ijk for k = (K, ℓ) is w_ℓ|K| (slot φ_i)(x_ℓ)(slot φ_j)(x_ℓ) — the discrete SGA term
 * with that rule is reproduced exactly.  N_q = n_dofs / n_cells; the rule is the
 * `quad` argument of egfem_tensor_build (n_points must equal N_q) or the default rule
 * with N_q points (2D: 1, 3, 6; 3D: 1, 4; 1D: 3).  The k-slot must be a value slot
 * (every form but CONV_K). */
typedef enum { EGFEM_P0 = 0, EGFEM_P1 = 1, EGFEM_P2 = 2, EGFEM_QUAD = 3 } egfem_family;

/* Trilinear forms, slot order (i = test, j = u-slot, k = w-slot):
 *   CONV_K : ∫ φ_i φ_j ∂x φ_k                 (BASELINE cfg1, 1D Burgers)
 *   CONV_J : ∫ φ_i (∂x+∂y)φ_j φ_k             (BASELINE cfg2/cfg5, 2D Burgers)
 *   PLAP   : ∫ ψ_k ∇φ_i·∇φ_j                  (K_a of PAPER.md L253, §5.5 p-Laplace)
 *   MASS3  : ∫ φ_i φ_j η_k                     (M of PAPER.md L327 / M_c̃ of L478)
 *   CONV_I : ∫ (∂x+∂y)φ_i φ_j φ_k             (N of PAPER.md L400)
 * (∂x+∂y) sums the first min(d,2) partial derivatives. */
typedef enum {
  EGFEM_FORM_CONV_K = 0,
  EGFEM_FORM_CONV_J = 1,
  EGFEM_FORM_PLAP = 2,
  EGFEM_FORM_MASS3 = 3,
  EGFEM_FORM_CONV_I = 4
} egfem_form;

/* Pointwise nonlinearities at the W-DOFs:
 *   IDENTITY        : w = u                     (W = V, GFEM, Π_u = I, L338)
 *   SQUARE          : w_k = u_k²                (W = V, L336 with Π = I)
 *   GRADPOW_P0      : w_K = ‖∇u_h|_K‖^{p−2}     (V = P1, W = P0, p-Laplace, L574/L582)
 *   P1_TO_P2_SQUARE : w = (Π_u u) ⊙ (Π_u u)     (V = P1, W = P2, Case 1, L336–338)
 *   MINSURF_P0      : w_K = (1 + ‖∇u_h|_K‖²)^{−1/2}  (V = P1, W = P0, minimal surface a(·), L605–611)
 *   RECIPROCAL      : w_k = 1 / (p + u_h(x_k))  (the biochemical c̃ = σ/(k+u) with σ = 1, k = p,
 *                     L520–535; W = V: at the nodes; W = P0 with V = P1: at the centroid,
 *                     u_h(x_K) = mean of the cell's vertex values)
 * With W = QUAD (V = P1) every kind but IDENTITY / P1_TO_P2_SQUARE is evaluated at the
 * quadrature points (Case 3, L133): GRADPOW_P0 / MINSURF_P0 (∇u_h is constant per cell),
 * RECIPROCAL and SQUARE (w = u_h(x_ℓ)²) at u_h(x_ℓ) = Σ_a λ_a(x_ℓ) u_a. */
typedef enum {
  EGFEM_INTERP_IDENTITY = 0,
  EGFEM_INTERP_SQUARE = 1,
  EGFEM_INTERP_GRADPOW_P0 = 2,
  EGFEM_INTERP_P1_TO_P2_SQUARE = 3,
  EGFEM_INTERP_MINSURF_P0 = 4,
  EGFEM_INTERP_RECIPROCAL = 5
} egfem_interp_kind;

/* PICARD: A = T·w.  NEWTON: J = T·w + (T·₂u)·D_u w, the Schur
 * complement of the block Jacobian D_zF̃ of PAPER.md L290 (reading C10). */
typedef enum { EGFEM_JAC_PICARD = 0, EGFEM_JAC_NEWTON = 1 } egfem_jac_mode;

/* Batched vector layouts: NODE_MAJOR U[i*B + p]; PAIR_MAJOR U[p*N + i]. */
typedef enum { EGFEM_LAYOUT_NODE_MAJOR = 0, EGFEM_LAYOUT_PAIR_MAJOR = 1 } egfem_layout;

/* Simplicial mesh Ω_h: host arrays. */
typedef struct {
  int32_t dim;            /* 1, 2 or 3 */
  int64_t n_vertices;
  const double* coords;   /* host, n_vertices*dim, row-major */
  int64_t n_cells;
  const int32_t* cells;   /* host, n_cells*(dim+1) vertex ids */
} egfem_mesh;

/* A DOF numbering of a space on the mesh.  cell_dofs == NULL means the canonical
 * numbering: P0 -> cell id, P1 -> vertex id (mesh cells), QUAD -> K·N_q + ℓ.  P2 (2D
 * only) needs an explicit table with local order (v0, v1, v2, m01, m12, m20). */
typedef struct {
  egfem_family family;
  int64_t n_dofs;
  const int32_t* cell_dofs; /* host, n_cells*n_local, or NULL (P0/P1 canonical) */
} egfem_space;

/* Quadrature rule in barycentric coordinates, weights summing to 1 (the |K|
 * factor is applied at assembly).  NULL = form default:
 * 1D 3-point Gauss; 2D centroid / 3-point degree-2 / 6-point degree-4 chosen by
 * the integrand's polynomial degree (degree-4 is capped: cfg5's degree-5
 * integrand is DEFINED by the 6-point rule, reading C3); 3D centroid / 4-point. */
typedef struct {
  int32_t n_points;
  const double* bary;     /* host, n_points*(dim+1) */
  const double* weights;  /* host, n_points */
} egfem_quad;

typedef struct egfem_tensor egfem_tensor; /* opaque; owns every device array */

/* ---------------------------------------------------------------- offline build
 * Assemble T_ijk = Σ_K ∫_K (slot_i φ_i)(slot_j φ_j)(slot_k η_k) over all cells,
 * keeping every structural triple (numeric zeros included, reading C7), summing
 * duplicates, in SPEC's canonical lexicographic (i,j,k) order.
 * The CSR pattern of the Jacobian is the union of element cliques over V-DOFs and
 * coincides with the (i,j) fibers of T.  Runs on `device`; returns after the
 * device work is complete.  Errors: INVALID_ARGUMENT (nulls, dim, cell_dofs out of
 * range), UNSUPPORTED (P2 outside 2D, a row longer than the kernel tile),
 * INDEX_OVERFLOW (N_f >= 2^28 for P0 W, nnz >= 2^32, n_dofs >= 2^31),
 * OUT_OF_MEMORY, CUDA.  *out is NULL on error. */
egfem_status egfem_tensor_build(const egfem_mesh* mesh, const egfem_space* V, const egfem_space* W,
                                egfem_form form, const egfem_quad* quad, egfem_dtype dtype,
                                int device, egfem_tensor** out);

/* Build from a user-supplied COO tensor (host arrays, any order, duplicates summed
 * in the given order).  The CSR pattern is the set of (i,j) fibers.  No mesh is
 * attached, so only IDENTITY / SQUARE interp and PICARD / IDENTITY- and
 * SQUARE-NEWTON Jacobians are available (they need W = V: n_f == n_u). */
egfem_status egfem_tensor_from_coo(int64_t n_u, int64_t n_f, int64_t nnz, const int32_t* i,
                                   const int32_t* j, const int32_t* k, const double* val,
                                   egfem_dtype dtype, int device, egfem_tensor** out);

egfem_status egfem_tensor_destroy(egfem_tensor* t);

/* Sizes.  Any output pointer may be NULL. */
egfem_status egfem_tensor_info(const egfem_tensor* t, int64_t* n_u, int64_t* n_f, int64_t* nnz,
                               int64_t* nnz_csr, egfem_dtype* dtype);

/* Borrowed device pointers to the CSR pattern (valid for the handle's lifetime):
 * row_ptr int64[N_u+1], col int32[nnz_csr], columns ascending within a row. */
egfem_status egfem_tensor_csr_pattern(const egfem_tensor* t, const int64_t** d_row_ptr,
                                      const int32_t** d_col);

/* Copy the canonical arrays to HOST buffers (NULL = skip):
 *   t_row_ptr int64[N_u+1], t_j int32[nnz], t_k int32[nnz], t_val (dtype)[nnz],
 *   csr_row_ptr int64[N_u+1], csr_col int32[nnz_csr],
 *   slot_ij int32[nnz]  CSR position of (i, t_j[e]),
 *   slot_ik int32[nnz]  CSR position of (i, t_k[e])  (W = V numbering only, else UNSUPPORTED),
 *   loc uint8[nnz]      bits 0-1: local index of i in cell t_k[e], bits 2-3: of t_j[e]
 *                       (P0 W only, else UNSUPPORTED).  Synchronous. */
egfem_status egfem_tensor_export(const egfem_tensor* t, int64_t* t_row_ptr, int32_t* t_j, int32_t* t_k,
                                 void* t_val, int64_t* csr_row_ptr, int32_t* csr_col, int32_t* slot_ij,
                                 int32_t* slot_ik, uint8_t* loc);

/* ---------------------------------------------------------------- per iteration
 * (1) w = f(Π_u u, Π_∇u ·₂ u) at every W-DOF.
 * u: device [N_u]; w: device [N_f].  chain (nullable; cell-wise W = P0 or QUAD only):
 * device [N_f*(d+1)], the pointwise D_u w of PAPER.md L292 for the cell K owning W-DOF k
 * (v_0..v_d its vertices), consumed by egfem_jacobian NEWTON with the same kind:
 *   RECIPROCAL, SQUARE:        chain[k*(d+1)+m] = ∂w_k/∂u_{v_m}, m = 0..d;
 *   GRADPOW_P0, MINSURF_P0:    chain[k*(d+1)] = w_k and chain[k*(d+1)+1+m] = ∂w_k/∂u_{v_m},
 *                              m = 0..d−1 (packed: ∂w_k/∂u_{v_d} = −Σ_{m<d} ∂w_k/∂u_{v_m},
 *                              exact because w depends on u through ∇u_h and Σ_m ∇λ_m = 0),
 *                              so the Newton kernel reads a cell's w and D_u w with one gather.  p > 1 required for GRADPOW_P0; p is k of RECIPROCAL (any value; p + u = 0
 * gives ±inf); p ignored otherwise.  At ∇u_h|_K = 0 and p < 4 the GRADPOW derivative is
 * taken as 0 (reading C11).  For GRADPOW_P0 / MINSURF_P0 with chain, w may be NULL: w_k is
 * then written only into the packed record chain[k*(d+1)] (one copy instead of two; the Newton
 * calls below read it from there). */
egfem_status egfem_interp(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u,
                          void* w, void* chain, egfem_stream_t stream);

/* (2) r_i = Σ_{(j,k)} T_ijk u_j w_k  (":" with A = u⊗w; L251).
 * u: [N_u], w: [N_f], r: [N_u], all device. */
egfem_status egfem_apply(const egfem_tensor* t, const void* u, const void* w, void* r,
                         egfem_stream_t stream);

/* (2b) the same for `batch` independent (u, w) pairs reusing each T nonzero:
 * R_p = T:(U_p ⊗ W_p).  Layout NODE_MAJOR: U[j*batch+p], W[k*batch+p], R[i*batch+p];
 * PAIR_MAJOR: U[p*N_u+j], ... (batch >= 1).  U may alias W (pairs (u, w = u): the u-slot
 * values are then taken from the W registers, and the compiled row groups evaluate the quadratic
 * form R_i = Σ_j u_j Σ_{k≥j} (T_ijk + T_ikj [k > j]) u_k from symmetrized patterns — the same sum
 * regrouped, within rounding of the unaliased call; EGFEM_GROUP_SYM=0 keeps the plain patterns).  W = V tensors with dense blocks run the
 * compiled row-group kernels for NODE_MAJOR (egfem_group.cu): the kernel variant for
 * (U aliases W, batch % 128 == 0) is NVRTC-compiled on its first use (a one-time host cost
 * of ~1 s, cached process-wide), and the call forks its small pattern classes onto the
 * handle's side streams and joins them back into `stream` with events (stream-ordered and
 * CUDA-graph capturable; concurrent callers enqueue one after the other). */
egfem_status egfem_apply_batched(const egfem_tensor* t, int32_t batch, egfem_layout layout,
                                 const void* U, const void* W, void* R, egfem_stream_t stream);

/* (3) Jacobian / Picard matrix values in the CSR pattern:
 *   PICARD              : A_ij = Σ_k T_ijk w_k
 *   NEWTON IDENTITY     : J = T·w + T·₂u                (∂w_k/∂u_m = δ_km)
 *   NEWTON SQUARE       : J = T·w + (T·₂u)·diag(2u)
 *   NEWTON RECIPROCAL   : J = T·w + (T·₂u)·diag(−1/(p+u)²)   (W = V)
 *   NEWTON cell-wise W  : J = T·w + (T·₂u)·D_u w, D_u w from `chain` (egfem_interp):
 *                         W = P0 or QUAD with GRADPOW_P0, MINSURF_P0, RECIPROCAL, (QUAD) SQUARE
 * u: [N_u] (NEWTON), w: [N_f], chain: [N_f*(d+1)] (P0-W NEWTON), csr_vals: [nnz_csr].
 * NEWTON with P1_TO_P2_SQUARE returns UNSUPPORTED.  w may be NULL in a NEWTON call of a packed
 * kind (GRADPOW_P0, MINSURF_P0, chain given) served by the cell-major kernels — they read w_K from
 * the packed record (egfem_kernel_name reports k_cell); otherwise NULL w is INVALID_ARGUMENT.
 * The same holds for egfem_apply_jacobian, egfem_apply_jacobian_rows and egfem_step. */
egfem_status egfem_jacobian(const egfem_tensor* t, egfem_jac_mode mode, egfem_interp_kind kind, double p,
                            const void* u, const void* w, const void* chain, void* csr_vals,
                            egfem_stream_t stream);

/* Fused (2)+(3): one pass over T produces r and csr_vals (same semantics and
 * arguments as egfem_apply + egfem_jacobian; results are bitwise identical to the
 * separate calls). */
egfem_status egfem_apply_jacobian(const egfem_tensor* t, egfem_jac_mode mode, egfem_interp_kind kind,
                                  double p, const void* u, const void* w, const void* chain, void* r,
                                  void* csr_vals, egfem_stream_t stream);

/* One Newton iteration's tensor work (PAPER.md L165–169 step (1), L183
 * and L290–292 steps (2)+(3)): exactly egfem_interp(t, kind, p, u, w, chain) followed by
 * egfem_apply_jacobian(t, NEWTON, kind, p, u, w, chain, r, csr_vals) — same arguments, same
 * checks, and w, chain, r, csr_vals bitwise identical to those two calls.  For the gradient
 * kinds (GRADPOW_P0, MINSURF_P0) on a mesh tensor with canonical P1 V / P0 W numbering whose
 * rows fit the cell-major kernel (and, 3D fp64, a 32-byte aligned chain) it runs as ONE
 * launch: warps take interp items (cells) and row items (rows) from one work sequence, a row
 * item starting once the records of its cells are written (release/acquire flags in the
 * handle), so the records are gathered from L2 while the interp of later cells overlaps.
 * The single-pass plan is opt-in — built with the tensor when EGFEM_STEP=1 is set — because
 * on B200 it measured slower than the two launches (both halves are bound by the SM
 * load/store pipe); otherwise, and for every other tensor / kind / a chain not
 * 32-byte aligned, it issues the two launches.  The single-pass state lives in the handle: calls on
 * one handle must be stream-ordered (not concurrent on two streams).  Stream-ordered and
 * CUDA-graph capturable. */
egfem_status egfem_step(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u, void* w,
                        void* chain, void* r, void* csr_vals, egfem_stream_t stream);

/* ---------------------------------------------------------------- bilinear GFEM forms
 * The matrix forms of PAPER.md L196–203 eq. (egfem_terms) and L402–409:
 *   M^c_ik = ∫ η_k φ_i   (the MASS3 tensor's form),   N^f_ik = ∫ η_k (∂x+∂y)φ_i   (CONV_I's),
 * the GFEM counterpart of a trilinear term in which the u-slot is absent.  For Lagrange V
 * (Σ_j φ_j ≡ 1) such a matrix is the u-slot contraction of the trilinear tensor with all ones,
 * B = T·₂1, and for W = V numbering its pattern is the tensor's CSR pattern (k runs over the
 * same element cliques as j).  The hot path of a GFEM term is then
 *   r = B f (egfem_csr_spmv),  J = B·diag(f'(u)) (egfem_bilinear_jacobian),
 * with f = w from egfem_interp (IDENTITY, SQUARE, RECIPROCAL).
 * egfem_bilinear_build: b_vals device [nnz_csr] ← B.  Needs W = V numbering whose T·₂u fits
 * the pattern (else DIMENSION_MISMATCH / UNSUPPORTED) and a value u-slot (MASS3, CONV_I,
 * CONV_K; CONV_J and PLAP differentiate it, T·₂1 = 0: UNSUPPORTED; a from_coo tensor is taken
 * as is; a partitioned local tensor: UNSUPPORTED).  Runs T·₂1 through the Newton kernel
 * (offline; two stream-ordered temporary vectors over the column space, cudaMallocAsync /
 * cudaFreeAsync: no synchronization, capturable in a CUDA graph). */
egfem_status egfem_bilinear_build(const egfem_tensor* t, void* b_vals, egfem_stream_t stream);

/* y = A x for any values `vals` [nnz_csr] on the tensor's CSR pattern (x: [N_u], y: [N_u], all
 * device, handle dtype); per-row sums in a fixed order. */
egfem_status egfem_csr_spmv(const egfem_tensor* t, const void* vals, const void* x, void* y,
                            egfem_stream_t stream);

/* GFEM Jacobian of r(u) = B f(u):  J_ik = B_ik f'(u_k)  (W = V; PAPER.md L290 with the
 * pointwise D_u f of L292): IDENTITY f' = 1, SQUARE 2u, RECIPROCAL −1/(p+u)².  b_vals, u, J
 * device ([nnz_csr], [N_u], [nnz_csr]); J is fully overwritten. */
egfem_status egfem_bilinear_jacobian(const egfem_tensor* t, const void* b_vals, egfem_interp_kind kind,
                                     double p, const void* u, void* csr_vals, egfem_stream_t stream);

/* ---------------------------------------------------------------- multi-GPU (row partition)
 * Split the rows of `global` into `nranks` contiguous ranges balanced by nnz and
 * build rank `rank`'s local tensor on `device`.  The local tensor addresses a
 * local vector of length n_local = halo_lo + owned + halo_hi laid out as global
 * indices [col_begin, col_end) (contiguous: the structured lexicographic numbering
 * makes the referenced columns one range; a non-contiguous range is still
 * correct, only larger).  Local W (P0) covers cells [w_begin, w_end) referenced by
 * the owned rows.  Outputs (host scalars, any may be NULL): row_begin/row_end
 * (owned global rows), col_begin/col_end (local u window), w_begin/w_end.  The local tensor
 * carries its own derived layouts (cell-major copy and packed row words, W = V transposes,
 * dense blocks and compiled row groups), so egfem_apply_batched on it — U / W the node-major
 * [col_begin, col_end) window, R its rows — is the row-partitioned batched action. */
egfem_status egfem_partition(const egfem_tensor* global, int32_t nranks, int32_t rank, int device,
                             egfem_tensor** local, int64_t* row_begin, int64_t* row_end,
                             int64_t* col_begin, int64_t* col_end, int64_t* w_begin, int64_t* w_end);

/* Pure host helper behind egfem_partition: nnz-balanced contiguous row split.
 * row_nnz_prefix: host int64[n_rows+1] (t_row_ptr); out_bounds: host int64[nranks+1]. */
egfem_status egfem_partition_rows(int64_t n_rows, const int64_t* row_nnz_prefix, int32_t nranks,
                                  int64_t* out_bounds);

/* Interior / boundary split of a tensor's work, for overlapping the u-halo exchange with
 * compute (§8(e); the step is PAPER.md L251/L290 restricted to a row range).  Rows
 * [row_lo, row_hi) read only owned u (columns, and for W = V the k indices, inside the
 * owned window [row_begin − col_begin, row_end − col_begin)), and interp work items
 * [w_lo, w_hi) read only owned u and cover every w those rows read.  So a rank can run
 *   interp_range(w_lo, w_hi) ; apply_jacobian_rows(row_lo, row_hi)      while u's halo is in flight,
 *   interp_range over the rest ; apply_jacobian_rows over the rest       after it has arrived,
 * and obtain bitwise the results of the whole-range calls.  Interp work items are W DOFs for
 * W = V and mesh cells for cell-wise W (P0 / QUAD / P2).  A global (unpartitioned) tensor
 * has no halo: its interior is everything.  An empty interior is returned as lo = hi = 0.
 * Outputs are host scalars (any may be NULL). */
egfem_status egfem_interior(const egfem_tensor* t, int64_t* row_lo, int64_t* row_hi, int64_t* w_lo,
                            int64_t* w_hi);

/* egfem_interp restricted to interp work items [lo, hi) (units as in egfem_interior; the
 * buffers are the whole-tensor u, w, chain).  0 <= lo <= hi <= n_items, else
 * INVALID_ARGUMENT. */
egfem_status egfem_interp_range(const egfem_tensor* t, egfem_interp_kind kind, double p, const void* u,
                                void* w, void* chain, int64_t lo, int64_t hi, egfem_stream_t stream);

/* egfem_apply_jacobian restricted to rows [row_lo, row_hi) (r and csr_vals are the
 * whole-tensor buffers; only those rows' entries are written).  A proper sub-range needs
 * one of the row-group kernels (rows of at most 512 nonzeros); the general tile path
 * returns UNSUPPORTED for it. */
egfem_status egfem_apply_jacobian_rows(const egfem_tensor* t, egfem_jac_mode mode, egfem_interp_kind kind,
                                       double p, const void* u, const void* w, const void* chain, void* r,
                                       void* csr_vals, int64_t row_lo, int64_t row_hi,
                                       egfem_stream_t stream);

/* Pure host helper behind egfem_interior: the longest run [lo, hi) of consecutive rows of a
 * CSR pattern (host int64 row_ptr[n_rows+1], int32 col) whose columns all lie in
 * [own_lo, own_hi); the first such run on ties, lo = hi = 0 when there is none. */
egfem_status egfem_interior_rows(int64_t n_rows, const int64_t* row_ptr, const int32_t* col, int64_t own_lo,
                                 int64_t own_hi, int64_t* lo, int64_t* hi);

/* Halo gather/scatter for non-contiguous exchanges: send_buf[q] = u_local[idx[q]],
 * u_local[idx[q]] = recv_buf[q] (device arrays, n entries, handle's dtype). */
egfem_status egfem_halo_pack(const egfem_tensor* local, const int32_t* d_idx, int64_t n,
                             const void* u_local, void* send_buf, egfem_stream_t stream);
egfem_status egfem_halo_unpack(const egfem_tensor* local, const int32_t* d_idx, int64_t n,
                               const void* recv_buf, void* u_local, egfem_stream_t stream);

/* Name of the kernel family `entry` dispatches to for this handle (0 = egfem_apply,
 * 1 = egfem_jacobian, 2 = egfem_apply_jacobian with (mode, kind, p), 3 = egfem_apply_batched
 * NODE_MAJOR, 4 = egfem_step with (kind, p), a 32-byte aligned chain assumed, 5 = egfem_interp
 * with kind: "k_interp_gradpow_geo" when the handle holds geometry classes), written
 * NUL-terminated into the host buffer buf[len] (truncated if short).
 * Used by bench.py to name the kernel its roofline line measures.  No launch.
 * INVALID_ARGUMENT on NULL t/buf, len = 0 or a bad entry; the Jacobian checks of
 * egfem_jacobian (without the pointer checks) for entries 1, 2 and 4. */
egfem_status egfem_kernel_name(const egfem_tensor* t, int32_t entry, egfem_jac_mode mode, egfem_interp_kind kind,
                               double p, char* buf, size_t len);

/* Diagnostic, no GPU needed: generates the compiled row-group kernel of the batched action
 * (egfem_group.cu) for one group pattern and compiles it with NVRTC for
 * sm_100a.  key[key_len] (host int32) serializes the pattern: n (stencil width), g (member
 * rows), then per member its fiber count and per fiber (a, count, b_1..b_count) — positions
 * in the n-point group stencil.  pairs_per_lane ∈ [1, 4]; fp64 if f64 else fp32.
 * EGFEM_OK when it compiles; INVALID_ARGUMENT for a malformed key; CUDA (detail in
 * egfem_last_error) when NVRTC fails.  EGFEM_GROUP_DUMP=<prefix> also writes the source and
 * the CUBIN. */
egfem_status egfem_group_compile(const int32_t* key, int32_t key_len, int32_t pairs_per_lane, int32_t f64);

/* Number of CUDA kernels this library launched (process-wide, all threads); used
 * by bench.py to report gpu_launches. */
uint64_t egfem_launch_count(void);

const char* egfem_status_string(egfem_status s);
const char* egfem_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* EGFEM_H */

/*
 * pfem.h — C-ABI of the B200-native PFEM hot path (arXiv 2601.03086, "Pretrained
 * Finite Element Method"): explicit finite-element differentiation of displacement
 * fields on P1 simplex meshes (T3 / T4), element and total strain energy, the
 * assembled internal force, the matrix-free tangent product and a warm-started CG.
 *
 * Citations are PAPER.md line numbers ("P:n") with their section; readings of
 * ambiguous passages are numbered R1.. in DESIGN.md §3.
 *
 * Conventions for every call
 *  - All array arguments are DEVICE pointers (CUDA global memory) unless a comment
 *    says "host".  The caller owns them (e.g. torch.empty on cuda); the library only
 *    allocates device memory inside pfem_mesh_prepare (the opaque plan, released by
 *    pfem_mesh_release) — never on the hot path.
 *  - `stream` is a cudaStream_t (passed as void*); every hot-path call is
 *    asynchronous on it.  pfem_mesh_prepare and pfem_cg synchronise the stream once
 *    to return host-side counts / reports.
 *  - Node fields are [S][N][d] (sample-major), contiguous inside a sample, with an
 *    explicit sample stride in ELEMENTS (not bytes).  Element arrays are SoA.
 *  - Floating point arrays have the dtype of the call (pfem_dtype).  Integers are
 *    int32.
 *  - Return value: PFEM_OK (0) or a negative pfem_status.  Argument / launch errors
 *    are returned synchronously; pfem_last_error() gives a message and
 *    pfem_last_error_index() the offending element / node (or -1).  Both are
 *    thread-local.  Data-dependent conditions of the asynchronous hot path (inverted
 *    Neo-Hookean elements, non-finite values) are reported through the optional
 *    device struct pfem_flags, written by the call.
 *  - No floating-point atomics: every sum has a fixed order, so two runs of the same
 *    call on the same inputs are bitwise identical.
 */
#ifndef PFEM_H
#define PFEM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFEM_ABI_VERSION 6

typedef enum {
    PFEM_OK = 0,
    PFEM_ERR_ARG = -1,           /* bad pointer / enum / size / connectivity out of range */
    PFEM_ERR_DEGENERATE = -2,    /* |det J_e| <= 64 eps_f64 prod |edges|; index = element */
    PFEM_ERR_INVERTED = -3,      /* reserved (NH inversion is reported via pfem_flags)    */
    PFEM_ERR_NOT_CONVERGED = -4, /* CG hit max_iter; x holds the partial iterate          */
    PFEM_ERR_BREAKDOWN = -5,     /* CG: p.Ap <= 0 (operator not SPD on the free DOFs)     */
    PFEM_ERR_CAPACITY = -6,      /* workspace / colour capacity too small                  */
    PFEM_ERR_CUDA = -7,          /* CUDA runtime error (message in pfem_last_error)        */
    PFEM_ERR_NOT_PREPARED = -8   /* mesh has no plan: call pfem_mesh_prepare first         */
} pfem_status;

typedef enum { PFEM_F32 = 0, PFEM_F64 = 1 } pfem_dtype;

/* Strain-energy density (§4.1; §4.2). */
typedef enum {
    PFEM_LINEAR = 0,     /* psi = 1/2 sigma:eps, sigma = 2 mu eps + lam tr(eps) I            */
    PFEM_NEOHOOKEAN = 1  /* psi = 1/2 lam (ln J)^2 - mu ln J + 1/2 mu (I1 - d)  (reading R2) */
} pfem_model;

/* Material parameter kind.  2-D runs are plane strain unless
 * PFEM_YOUNG_POISSON_PLANE_STRESS (lam* = 2 mu lam / (lam + 2 mu)) — reading R1. */
typedef enum {
    PFEM_LAME = 0,                       /* p0 = mu, p1 = lambda */
    PFEM_YOUNG_POISSON = 1,              /* p0 = E,  p1 = nu      */
    PFEM_YOUNG_POISSON_PLANE_STRESS = 2  /* p0 = E,  p1 = nu      */
} pfem_param;

/* Deterministic assembly of element contributions into nodes (north star: never float
 * atomics on the reported path). */
typedef enum {
    PFEM_ASSEMBLE_CSR = 0,    /* block-partitioned CSR gather: every node sums its (element,
                                 slot) entries in ascending element order, segment by segment
                                 over the element blocks touching it        */
    PFEM_ASSEMBLE_COLOUR = 1  /* colour-ordered scatter: one pass per colour of the greedy
                                 element colouring, one non-atomic read-modify-write per
                                 (element, slot)                                              */
} pfem_assembly;

typedef enum {
    PFEM_ORDER_INPUT = 0,          /* blocks of consecutive input elements                      */
    PFEM_ORDER_LOCALITY = 1,       /* blocks of consecutive elements in Morton order of their
                                      centroids, inside each part (fewer nodes shared by blocks) */
    PFEM_ORDER_AUTO = 2            /* whichever of the two gives fewer (block, node) occurrences  */
} pfem_elem_order;

/* Element geometry of the CSR-mode element kernels (SURVEY §8(f) row f4 variant). */
typedef enum {
    PFEM_GEOMETRY_STORED = 0,      /* read grad / vol prepared by pfem_mesh_prepare                 */
    PFEM_GEOMETRY_ON_THE_FLY = 1   /* form grad N_a and V_e in fp64 from `coords` inside the element
                                      pass (same formula as prepare; fewer HBM bytes, more ALU).
                                      Applies to PFEM_ASSEMBLE_CSR energy / residual / tangent and
                                      the solvers built on them; COLOUR mode reads grad / vol      */
} pfem_geometry;

/* Element family (SURVEY §8(f) row f4 for the quadrilaterals). */
typedef enum {
    PFEM_ELEM_SIMPLEX = 0,   /* P1 triangles (dim 2) / tetrahedra (dim 3), one-point rule (reading R4)  */
    PFEM_ELEM_Q4 = 1,        /* bilinear quadrilateral, 2 x 2 Gauss (dim 2; beam P:774)              */
    PFEM_ELEM_Q8 = 2         /* serendipity quadrilateral, 3 x 3 Gauss (dim 2; Cook P:846); nodes:
                                4 corners counter-clockwise, then midsides of edges 01, 12, 23, 30   */
} pfem_elem_type;

typedef struct pfem_plan pfem_plan;   /* opaque, library-owned device data */

/* Mesh descriptor.  Inputs are set by the caller; pfem_mesh_prepare fills the outputs. */
typedef struct {
    /* ---- inputs ---- */
    int32_t dim;                   /* 2 (T3) or 3 (T4)                                          */
    int32_t n_nodes, n_elems;
    int32_t n_parts;               /* >= 1: independent meshes concatenated (config 5)          */
    int32_t dtype;                 /* pfem_dtype of grad / vol and of every field call          */
    int32_t block_elems;           /* assembly block size (elements); 0 = library default       */
    int32_t elem_order;            /* assembly element order (pfem_elem_order): the plan may visit
                                      elements in a locality order; results are unchanged up to
                                      rounding and are reported in input element order           */
    int32_t geometry;              /* pfem_geometry; may change between calls (coords must stay valid) */
    int32_t elem_type;             /* pfem_elem_type; conn is [n_elems][nodes per element].  Q4 / Q8:
                                      dim 2, CSR assembly only, no Jacobi / heat / pretraining calls;
                                      grad / vol are not written (the Gauss-point geometry lives in
                                      the plan)                                                     */
    const double* coords;          /* [n_nodes][dim], float64 always                             */
    const int32_t* conn;           /* [n_elems][dim+1], node ids in [0, n_nodes)                 */
    const int32_t* part_elem;      /* [n_parts+1] element offsets (device), NULL if n_parts == 1 */
    const int32_t* part_node;      /* [n_parts+1] node offsets (device),    NULL if n_parts == 1 */
    /* ---- outputs of pfem_mesh_prepare (device, caller-allocated) ---- */
    void* grad;                    /* [dim*dim][n_elems] SoA: grad[(a*dim + j)*E + e] = dN_{a+1}/dX_j,
                                      rows of J_e^{-1}, J_e = [X_1-X_0 | .. | X_d-X_0]
                                      (P1 shape functions, App. B; dN_0 = -sum)      */
    void* vol;                     /* [n_elems] V_e = |det J_e| / d!                             */
    int32_t* csr_ptr;              /* [n_nodes+1] node -> (element, slot) CSR row offsets       */
    int32_t* csr_ent;              /* [(dim+1)*n_elems] e*(dim+1)+slot, ascending per row (R12)  */
    int32_t* colour;               /* [n_elems] greedy first-fit colour in element order (R12)   */
    int32_t* colour_elems;         /* [n_elems] elements sorted by (colour, element)             */
    int32_t* colour_ptr;           /* [max_colours+1] offsets into colour_elems                  */
    int32_t max_colours;           /* capacity of colour_ptr - 1 (<= 128)                        */
    /* ---- host outputs of pfem_mesh_prepare ---- */
    int32_t n_colours;
    int32_t n_negative;            /* elements with det J_e < 0 (valid; gradients are exact)    */
    int32_t n_blocks;              /* assembly blocks of the plan                                */
    int32_t n_occ;                 /* (block, node) occurrences of the plan                      */
    pfem_plan* plan;               /* set by prepare; free with pfem_mesh_release                */
} pfem_mesh;

/* Material: per-element parameters with an element stride each (stride 0 = uniform).
 * Arrays have the call's dtype. */
typedef struct {
    int32_t model;                 /* pfem_model */
    int32_t kind;                  /* pfem_param */
    const void* p0;
    const void* p1;
    int64_t stride0, stride1;      /* in elements; 0 broadcasts p0[0] / p1[0] */
} pfem_material;

/* Device-side report of data-dependent conditions, written (not accumulated) by every
 * hot-path call that receives it. */
typedef struct {
    int32_t n_inverted;            /* Neo-Hookean elements with J = det F <= 0 (NaN energy)  */
    int32_t first_inverted;        /* lowest such element id, or -1                           */
    int32_t n_nonfinite;           /* elements whose energy density or stress is not finite    */
    int32_t reserved;
} pfem_flags;

/* ---------------------------------------------------------------------------------
 * Mesh preparation (one-time per mesh; §8 row a1).
 * Computes, on the GPU: shape-function gradients and volumes (fp64 arithmetic, stored
 * in m->dtype), the node->(element,slot) CSR, the greedy element colouring and its
 * colour-sorted list, and the assembly plan (element blocks, block-local CSR, node
 * occurrences).  Errors: PFEM_ERR_ARG (sizes, null pointers, conn out of range, index
 * = element), PFEM_ERR_DEGENERATE (index = lowest degenerate element),
 * PFEM_ERR_CAPACITY (more than max_colours colours).  Synchronises `stream`.
 * Re-preparing a mesh that already has a plan releases the old plan first.
 * --------------------------------------------------------------------------------- */
pfem_status pfem_mesh_prepare(pfem_mesh* m, void* stream);
void pfem_mesh_release(pfem_mesh* m);

/* Device copies of the plan arrays, for tests (host pointers to fill, each may be NULL).
 * Sizes: blk_elem [n_blocks+1] (plan positions), blk_occ [n_blocks+1], occ_node [n_occ]
 * (node id | kind bits 29..30), occ_ent_ptr [n_occ+1], loc_ent [(dim+1)*n_elems] (uint16),
 * elem_perm [n_elems] (position -> input element id). */
pfem_status pfem_plan_export(const pfem_mesh* m, int32_t* blk_elem, int32_t* blk_occ,
                             int32_t* occ_node, int32_t* occ_ent_ptr, uint16_t* loc_ent,
                             int32_t* elem_perm);

/* Bytes of the per-call workspace of pfem_energy / pfem_residual / pfem_tangent_apply
 * for `n_samples` fields.  The workspace must be ZERO-FILLED before its first use; the
 * library keeps it consistent afterwards.  Calls sharing a workspace must be ordered on
 * one stream. */
size_t pfem_workspace_bytes(const pfem_mesh* m, int32_t n_samples);

/* Material conversion (E, nu) -> (mu, lambda)  (§8 K8).  out arrays [n]. */
pfem_status pfem_lame(int32_t dtype, int32_t kind, int64_t n, const void* p0, int64_t stride0,
                      const void* p1, int64_t stride1, void* mu, void* lam, void* stream);

/* ---------------------------------------------------------------------------------
 * Energy (and optionally the fused residual) of S displacement fields on one mesh.
 * §8 rows a2-a5.  Per element e and sample s:
 *   H = sum_{a=1..d} (u_{v_a} - u_{v_0}) (x) grad N_a,  F = I + H,
 *   W_e = V_e psi(H),   totals[s][k] = sum_{e in part k} W_e  - [f_ext given] sum_{n in part k} f_ext,n . u_n
 *   (the potential energy Pi = W - f.u of P:518-524 when f_ext is given; reading R6)
 * and, if residual != NULL, the internal force f_int (App. B):
 *   residual[s][n] = sum_{(e,a): v_a(e) = n} V_e P_e grad N_a
 * with P the first Piola-Kirchhoff stress (linear: sigma).  The solver residual is
 * f_int - f_ext (reading R7).
 * Arguments:
 *   u            [S][N][d], element stride `sample_stride` between samples
 *   f_ext        nullable [N][d] (shared by all samples)
 *   elem_energy  nullable [S][E]
 *   totals       [S][n_parts]
 *   residual     nullable [S][N][d] (same sample stride as u)
 *   mode         pfem_assembly
 *   flags        nullable device pfem_flags
 *   ws, ws_bytes per-call workspace (pfem_workspace_bytes), zero-filled before first use
 * --------------------------------------------------------------------------------- */
pfem_status pfem_energy(const pfem_mesh* m, const pfem_material* mat, int32_t n_samples,
                        const void* u, int64_t sample_stride, const void* f_ext,
                        void* elem_energy, void* totals, void* residual, int32_t mode,
                        pfem_flags* flags, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * Pretraining loss and its gradient w.r.t. the network output: the
 * energy-based loss of P:518-541 (linear) / P:700-723 (Neo-Hookean) through the hard-BC
 * ansatz u = (x/L) (.) H_theta, batch-averaged as in Eq. 2 over samples and parts
 * (reading R28):
 *   u = phi (.) H                                   (phi NULL: u = H, no copy)
 *   totals[s][k] = Pi_{s,k} = W_{s,k}(u) - sum_{n in part k} f_ext,n . u_n
 *   *loss = sum_{s,k} Pi_{s,k} / (S K)              (device double, row order)
 *   grad[s][n] = phi_n (.) (f_int(u)_n - f_ext,n) / (S K)
 * Arguments:
 *   H        [S][N][d] network output, sample stride `sample_stride`
 *   phi      nullable [N][d] ansatz multiplier (e.g. x/L per component, or the distance to a
 *            clamped edge broadcast over components), shared by all samples
 *   f_ext    nullable [N][d]
 *   u        [S][N][d] output (the ansatz field), required iff phi != NULL
 *   totals   [S][n_parts];  grad [S][N][d];  loss: device double
 *   mode, flags, ws, ws_bytes: as pfem_energy (same workspace)
 * Launches: the ansatz (if phi), the fused energy + residual of pfem_energy, the epilogue.
 * --------------------------------------------------------------------------------- */
pfem_status pfem_pretrain_loss(const pfem_mesh* m, const pfem_material* mat, int32_t n_samples,
                               const void* H, int64_t sample_stride, const void* phi,
                               const void* f_ext, void* u, void* totals, void* grad, double* loss,
                               int32_t mode, pfem_flags* flags, void* ws, size_t ws_bytes,
                               void* stream);

/* ---------------------------------------------------------------------------------
 * Steady heat conduction, the paper's scalar example (energy
 * form P:249-284), one DOF per node on the prepared mesh (geometry and CSR of
 * pfem_mesh_prepare):
 *   grad T_e = sum_a T_a grad N_a,   W_e = 1/2 k_e V_e |grad T_e|^2
 *   totals[s][k] = sum_{e in part k} W_e - sum_{n in part k} f_n T_n
 *   flux[s][n]   = sum_{(e,a): v_a(e) = n} k_e V_e grad T_e . grad N_a   (= dW/dT_n; the
 *                  operator is linear, so flux(v) is also K v)
 * Arguments:
 *   k            conductivity per element (k_stride 1) or uniform (k_stride 0), the mesh dtype
 *   T            [S][N], element stride `sample_stride` between samples
 *   f_nodal      nullable [N] consistent nodal loads of the source and the boundary flux
 *   elem_energy  nullable [S][E]; required when totals is given
 *   totals       nullable [S][n_parts];  flux: nullable [S][N]
 *   ws, ws_bytes per-call workspace (pfem_heat_workspace_bytes): the totals' slice sums and
 *                the fluxes' CSR-ordered entry buffer; may be NULL without totals (the fluxes
 *                then re-form each element per CSR entry, same summation order).  The
 *                workspace caches the CSR entry positions of the prepared mesh it was last
 *                used with (keyed by the plan; recomputed when the mesh changes); it must be
 *                ZERO-FILLED before its first use
 * Sums in fixed order (per part: 64 fixed slices, each a CTA tree, then the slices in order;
 * per node: CSR order); asynchronous on `stream`.
 * --------------------------------------------------------------------------------- */
/* options: PFEM_HEAT_GEOMETRY_ON_THE_FLY forms grad N_a and V_e in fp64 from the mesh
 * coordinates inside the element pass (with a workspace and fluxes requested) instead of
 * reading the prepared gradients and volumes (SURVEY §8(f) row f4 variant) */
#define PFEM_HEAT_GEOMETRY_ON_THE_FLY 1
size_t pfem_heat_workspace_bytes(const pfem_mesh* m, int32_t n_samples);
pfem_status pfem_heat(const pfem_mesh* m, const void* k, int64_t k_stride, int32_t n_samples,
                      const void* T, int64_t sample_stride, const void* f_nodal, void* elem_energy,
                      void* totals, void* flux, int32_t options, void* ws, size_t ws_bytes,
                      void* stream);

/* Internal force only (no energy arithmetic), see pfem_energy. */
pfem_status pfem_residual(const pfem_mesh* m, const pfem_material* mat, int32_t n_samples,
                          const void* u, int64_t sample_stride, void* residual, int32_t mode,
                          pfem_flags* flags, void* ws, size_t ws_bytes, void* stream);

/* Matrix-free tangent K(u) v (App. B; §8 row a6):
 *   linear: dP = 2 mu sym(dH) + lam tr(dH) I            (u ignored, may be NULL)
 *   NH:     dP = mu dH + (mu - lam ln J) F^-T dH^T F^-T + lam tr(F^-1 dH) F^-T,  F = I + grad u
 *   (Kv)_n = sum_{(e,a): v_a(e)=n} V_e dP_e grad N_a,  dH = sum_a (v_{v_a} - v_{v_0}) (x) grad N_a
 * With dirichlet_mask (nullable [N*d] uint8, 1 = constrained DOF) the call applies the
 * SPD masked operator (I-M) K (I-M) v + M v (reading R9).
 * u, v, Kv: [S][N][d] with the same sample stride. */
pfem_status pfem_tangent_apply(const pfem_mesh* m, const pfem_material* mat, int32_t n_samples,
                               const void* u, const void* v, void* Kv, int64_t sample_stride,
                               const uint8_t* dirichlet_mask, int32_t mode, pfem_flags* flags,
                               void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * Warm-started conjugate gradient (App. B; warm start P:395-417; skip rule
 * P:419-423; §8 row a7).  Solves A x = b on one field (S = 1):
 *   A = (I-M) K(u_state) (I-M) + M,   b = (I-M)(rhs - K x_D) + M x0,   x_D = M x0
 * Hestenes-Stiefel CG, unpreconditioned (reading R9), stop when the recurrence residual
 * satisfies ||r_k|| < tol ||b_free|| (strict, relative; reading R8).  iterations = number
 * of A p products (R11); 0 if x0 already satisfies the test.
 *   u_state  nullable [N][d] NH linearisation point (NULL for linear)
 *   rhs      [N][d] external force f_ext
 *   mask     nullable [N*d]
 *   x        in: x0 (constrained entries = prescribed values); out: solution / partial
 *   history  nullable device double [max_iter+1]: ||r_k|| / ||b_free||
 *   report   host
 * Iteration: in CSR mode on simplex meshes the pipelined form of SURVEY §8(f) row f3 (reading
 * R34): the element kernel forms p = z + beta p while staging p, kernel B forms p.q and alpha,
 * one update pass forms x, r, r.r and beta — 3 launches, the iterates of the unfused loop.
 * COLOUR mode and Q4 / Q8 meshes run the unfused 4-launch loop.  32 iterations are captured in a
 * CUDA graph, cached per host thread for calls with the same arrays, workspace and options.
 * Synchronises `stream`.  Returns PFEM_OK, PFEM_ERR_NOT_CONVERGED or PFEM_ERR_BREAKDOWN
 * (report filled in all three cases).
 * --------------------------------------------------------------------------------- */
typedef struct {
    int32_t iterations;
    int32_t converged;
    int32_t status;
    int32_t reserved;
    double rel_res0;           /* ||r_0|| / ||b_free||                          */
    double rel_res_final;      /* recurrence residual at exit                   */
    double true_rel_res_final; /* ||b - A x|| / ||b_free|| recomputed at exit   */
    double bnorm;              /* ||b_free||                                    */
} pfem_cg_report;

size_t pfem_cg_workspace_bytes(const pfem_mesh* m);
pfem_status pfem_cg(const pfem_mesh* m, const pfem_material* mat, const void* u_state,
                    const void* rhs, const uint8_t* mask, void* x, double tol, int32_t max_iter,
                    int32_t mode, double* history, pfem_cg_report* report, void* ws,
                    size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * Jacobi preconditioning.  The paper names preconditioning as the
 * complement of the warm start for cutting CG iterations (§5.5); DESIGN.md
 * reading R27 fixes the preconditioner (Jacobi) and the algorithm.
 *
 * pfem_tangent_diag: diag [N][d] of A = (I-M) K(u_state) (I-M) + M, 1 on constrained DOFs.
 *   Per DOF (n, i) the sum, over the (e, a) entries of node n in ascending CSR order (R12), of
 *     V_e [mu |grad N_a|^2 + c ((F^-T grad N_a)_i)^2],  c = lam + mu - lam ln J   (NH)
 *   (linear: F = I, c = lam + mu): the diagonal of the element tangent dP/dF of
 *   App. B P:1104-1115 contracted with grad N_a on both sides.
 *   u_state  nullable [N][d] (required for Neo-Hookean)
 *   mask     nullable [N*d]
 *   Asynchronous on `stream`; no workspace.
 *
 * pfem_pcg: pfem_cg with a preconditioner M (precond = PFEM_PRECOND_NONE: identical to
 *   pfem_cg; PFEM_PRECOND_JACOBI: M = diag(A), M^-1_k = 1/diag_k, 1 where diag_k <= 0):
 *     r0 = b - A x0, z = M^-1 r, p = z, rho = r.z;  per iteration q = A p, alpha = rho / p.q,
 *     x += alpha p, r -= alpha q, stop when ||r|| < tol ||b_free|| (unchanged, R8),
 *     z = M^-1 r, beta = (r.z)_new / rho, p = z + beta p.
 *   Same arguments, workspace (pfem_cg_workspace_bytes), report and errors as pfem_cg.
 * --------------------------------------------------------------------------------- */
typedef enum { PFEM_PRECOND_NONE = 0, PFEM_PRECOND_JACOBI = 1 } pfem_precond;

pfem_status pfem_tangent_diag(const pfem_mesh* m, const pfem_material* mat, const void* u_state,
                              void* diag, const uint8_t* mask, void* stream);
pfem_status pfem_pcg(const pfem_mesh* m, const pfem_material* mat, const void* u_state,
                     const void* rhs, const uint8_t* mask, int32_t precond, void* x, double tol,
                     int32_t max_iter, int32_t mode, double* history, pfem_cg_report* report,
                     void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * Newton-Raphson for the nonlinear (Neo-Hookean) warm-start stage (App. B P:1118-1139,
 * warm start U_0 = U^NO P:1141-1166; §8(f) row f1).  One load step, dead loads (K^ext = 0):
 *   r(U_k) = f_int(U_k) - f_ext  on free DOFs;  stop when ||r||_2 <= tol  (absolute)
 *   dU solves K(U_k) dU = -r with the masked CG of pfem_cg (x0 = 0, relative tolerance
 *   cg_tol, at most cg_max_iter products); constrained DOFs keep their values in u
 *   U_{k+1} = U_k + dU
 *   u        in: U_0 (constrained entries = prescribed values); out: the last iterate [N][d]
 *   f_ext    nullable [N][d]
 *   history  nullable HOST double [max_newton+1]: ||r(U_k)||
 *   report   host; iterations = Newton steps taken (0 if U_0 already satisfies the test)
 * Synchronises `stream` once per Newton step.  Returns PFEM_OK, PFEM_ERR_NOT_CONVERGED
 * (max_newton reached or non-finite residual) or PFEM_ERR_BREAKDOWN (indefinite tangent
 * met by the inner CG); the report is filled in every case.
 * --------------------------------------------------------------------------------- */
typedef struct {
    int32_t iterations;
    int32_t converged;
    int32_t status;            /* 0 converged, 1 max_newton, 2 CG breakdown, 3 non-finite    */
    int32_t cg_iterations;     /* inner CG products summed over the Newton steps             */
    double res0;               /* ||r(U_0)||                                                 */
    double res_final;          /* ||r|| of the last iterate                                  */
} pfem_newton_report;

size_t pfem_newton_workspace_bytes(const pfem_mesh* m);
pfem_status pfem_newton(const pfem_mesh* m, const pfem_material* mat, void* u, const void* f_ext,
                        const uint8_t* mask, double tol, int32_t max_newton, double cg_tol,
                        int32_t cg_max_iter, int32_t mode, double* history,
                        pfem_newton_report* report, void* ws, size_t ws_bytes, void* stream);

/* Diagnostics */
const char* pfem_last_error(void);
int64_t pfem_last_error_index(void);
int32_t pfem_abi_version(void);
/* number of kernel launches issued by this thread since the last reset (bench evidence) */
int64_t pfem_launch_count(int32_t reset);
/* Measured FMA-pipe peak of the current device (the denominators of the ALU
 * floors; not on the hot path).  kind 0: fp32 FFMA, 1: fp32 packed FFMA2 (two FMAs per lane
 * and issue slot), 2: fp64 DFMA; every thread of a resident grid runs 8 independent chains of
 * `iters` dependent FMAs from register operands.  Writes lane FMAs per second (x 2 = flop/s)
 * to the HOST double *lane_fma_per_s.  Synchronous: it allocates 32 bytes of device memory,
 * times 4 launches with CUDA events on `stream` and waits for them.
 * Errors: PFEM_ERR_ARG (kind, iters, null result), PFEM_ERR_CUDA. */
pfem_status pfem_fma_peak(int32_t kind, int32_t iters, double* lane_fma_per_s, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PFEM_H */

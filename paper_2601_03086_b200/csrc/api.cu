// api.cu — the extern "C" boundary (include/pfem.h): argument validation, thread-local
// errors, dispatch to the kernels.  No arithmetic of the method happens on the host.
#include <cstdio>
#include <cstring>

#include "launch.cuh"

namespace pfem {

static thread_local std::string g_err;
static thread_local int64_t g_err_index = -1;
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg, int64_t index) {
    g_err = msg;
    g_err_index = index;
}

pfem_status cuda_status(cudaError_t e, const char* what) {
    set_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
    return PFEM_ERR_CUDA;
}

void count_launch(int n) { g_launches += n; }

pfem_status prepare_impl(pfem_mesh* m, cudaStream_t s);
void release_impl(pfem_mesh* m);
size_t cg_ws_bytes(const Plan& P, int dtype);
size_t newton_ws_bytes(const Plan& P, int dtype);
pfem_status run_newton(const pfem_mesh* m, const pfem_material* mat, void* u, const void* fext, const uint8_t* mask,
                       double tol, int max_newton, double cg_tol, int cg_max_iter, int mode, double* history,
                       pfem_newton_report* rep, void* ws, cudaStream_t s);
pfem_status run_cg(const pfem_mesh* m, const pfem_material* mat, const void* u_state, const void* rhs,
                   const uint8_t* mask, void* x, double tol, int max_iter, int mode, double* history,
                   pfem_cg_report* rep, void* ws, cudaStream_t s, int precond);
pfem_status run_tangent_diag(const pfem_mesh* m, const pfem_material* mat, const void* u, const uint8_t* mask,
                             int invert, void* out, cudaStream_t s);
pfem_status run_heat(const pfem_mesh* m, const void* k, int64_t kstride, int S, const void* Tf, int64_t sstride,
                     const void* f, void* W, void* totals, void* r, void* ws, int otf, cudaStream_t s);
size_t heat_ws_bytes(const pfem_mesh* m, int S);
pfem_status run_pretrain_stage(const pfem_mesh* m, int S, int64_t sstride, const void* H, const void* phi, void* u,
                               int stage, const void* f_ext, void* grad, const void* totals, double* loss,
                               cudaStream_t s);

template <class T>
__global__ void k_lame(int64_t n, int kind, const T* p0, int64_t s0, const T* p1, int64_t s1, T* mu, T* lam) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    T m, l;
    lame_of<T>(kind, p0[i * s0], p1[i * s1], m, l);
    mu[i] = m;
    lam[i] = l;
}

static pfem_status check_mesh(const pfem_mesh* m, bool need_plan) {
    (void)cudaGetLastError();   // clear stale non-sticky runtime errors of earlier calls
    if (!m) { set_error("mesh is NULL"); return PFEM_ERR_ARG; }
    if (m->dim != 2 && m->dim != 3) { set_error("dim must be 2 or 3"); return PFEM_ERR_ARG; }
    if (m->dtype != PFEM_F32 && m->dtype != PFEM_F64) { set_error("bad dtype"); return PFEM_ERR_ARG; }
    if (m->n_nodes <= 0 || m->n_elems <= 0 || m->n_parts <= 0) {
        set_error("n_nodes, n_elems and n_parts must be positive");
        return PFEM_ERR_ARG;
    }
    if (need_plan && !m->plan) { set_error("mesh not prepared"); return PFEM_ERR_NOT_PREPARED; }
    return PFEM_OK;
}

static pfem_status check_mat(const pfem_material* mat) {
    if (!mat || !mat->p0 || !mat->p1) { set_error("material arrays are NULL"); return PFEM_ERR_ARG; }
    if (mat->model != PFEM_LINEAR && mat->model != PFEM_NEOHOOKEAN) { set_error("bad model"); return PFEM_ERR_ARG; }
    if (mat->kind < 0 || mat->kind > 2) { set_error("bad material kind"); return PFEM_ERR_ARG; }
    if (mat->stride0 < 0 || mat->stride1 < 0) { set_error("negative material stride"); return PFEM_ERR_ARG; }
    return PFEM_OK;
}

static pfem_status run(const Call& c) {
    const int D = c.m->dim;
    if (D == 2) return c.m->dtype == PFEM_F32 ? run_assemble<2, float>(c) : run_assemble<2, double>(c);
    return c.m->dtype == PFEM_F32 ? run_assemble<3, float>(c) : run_assemble<3, double>(c);
}

static pfem_status common_checks(const pfem_mesh* m, const pfem_material* mat, int S, int64_t sstride, int mode,
                                 void* ws, size_t ws_bytes) {
    pfem_status st = check_mesh(m, true);
    if (st) return st;
    if ((st = check_mat(mat))) return st;
    if (S <= 0) { set_error("n_samples must be positive"); return PFEM_ERR_ARG; }
    if (sstride < (int64_t)m->n_nodes * m->dim && S > 1) {
        set_error("sample_stride smaller than n_nodes*dim");
        return PFEM_ERR_ARG;
    }
    if (mode != PFEM_ASSEMBLE_CSR && mode != PFEM_ASSEMBLE_COLOUR) { set_error("bad assembly mode"); return PFEM_ERR_ARG; }
    if (m->elem_type != PFEM_ELEM_SIMPLEX && mode != PFEM_ASSEMBLE_CSR) {
        set_error("quadrilateral meshes assemble in CSR mode only");
        return PFEM_ERR_ARG;
    }
    if (m->geometry != PFEM_GEOMETRY_STORED && m->geometry != PFEM_GEOMETRY_ON_THE_FLY) {
        set_error("bad geometry option");
        return PFEM_ERR_ARG;
    }
    if (m->geometry == PFEM_GEOMETRY_ON_THE_FLY && !m->coords) {
        set_error("on-the-fly geometry needs coords");
        return PFEM_ERR_ARG;
    }
    if (!ws) { set_error("workspace is NULL"); return PFEM_ERR_ARG; }
    const Plan* P = reinterpret_cast<const Plan*>(m->plan);
    if (ws_bytes < ws_layout(*P, S, m->dtype == PFEM_F64 ? 8 : 4).total) {
        set_error("workspace too small (pfem_workspace_bytes)");
        return PFEM_ERR_CAPACITY;
    }
    return PFEM_OK;
}

}  // namespace pfem

using namespace pfem;

extern "C" {

const char* pfem_last_error(void) { return g_err.c_str(); }
int64_t pfem_last_error_index(void) { return g_err_index; }
int32_t pfem_abi_version(void) { return PFEM_ABI_VERSION; }
int64_t pfem_launch_count(int32_t reset) {
    int64_t v = g_launches;
    if (reset) g_launches = 0;
    return v;
}

pfem_status pfem_mesh_prepare(pfem_mesh* m, void* stream) {
    pfem_status st = check_mesh(m, false);
    if (st) return st;
    if (!m->coords || !m->conn || !m->grad || !m->vol || !m->csr_ptr || !m->csr_ent || !m->colour ||
        !m->colour_elems || !m->colour_ptr) {
        set_error("prepare: NULL input or output array");
        return PFEM_ERR_ARG;
    }
    if (m->n_parts > 1 && (!m->part_elem || !m->part_node)) {
        set_error("prepare: part offsets required when n_parts > 1");
        return PFEM_ERR_ARG;
    }
    if (m->n_nodes >= (1 << 29)) { set_error("n_nodes >= 2^29 not supported"); return PFEM_ERR_ARG; }
    if ((int64_t)m->n_elems * (m->dim + 1) >= INT32_MAX) { set_error("too many elements"); return PFEM_ERR_ARG; }
    if (m->max_colours < 1 || m->max_colours > 128) { set_error("max_colours must be in [1, 128]"); return PFEM_ERR_ARG; }
    if (m->block_elems < 0) { set_error("block_elems must be >= 0"); return PFEM_ERR_ARG; }
    if (m->elem_order < 0 || m->elem_order > 2) { set_error("elem_order must be 0, 1 or 2"); return PFEM_ERR_ARG; }
    if (m->geometry < 0 || m->geometry > 1) { set_error("geometry must be 0 or 1"); return PFEM_ERR_ARG; }
    if (m->elem_type < PFEM_ELEM_SIMPLEX || m->elem_type > PFEM_ELEM_Q8) { set_error("bad elem_type"); return PFEM_ERR_ARG; }
    if (m->elem_type != PFEM_ELEM_SIMPLEX && m->dim != 2) { set_error("Q4 / Q8 elements need dim 2"); return PFEM_ERR_ARG; }
    if (m->dim == 3 && ((uintptr_t)m->conn & 15)) { set_error("conn must be 16-byte aligned for dim 3"); return PFEM_ERR_ARG; }
    if (m->plan) release_impl(m);
    return prepare_impl(m, (cudaStream_t)stream);
}

void pfem_mesh_release(pfem_mesh* m) { release_impl(m); }

pfem_status pfem_plan_export(const pfem_mesh* m, int32_t* blk_elem, int32_t* blk_occ, int32_t* occ_node,
                             int32_t* occ_ent_ptr, uint16_t* loc_ent, int32_t* elem_perm) {
    pfem_status st = check_mesh(m, true);
    if (st) return st;
    const Plan* P = reinterpret_cast<const Plan*>(m->plan);
    if (P->elem_type != PFEM_ELEM_SIMPLEX) { set_error("quadrilateral meshes have no block plan"); return PFEM_ERR_ARG; }
    cudaError_t e = cudaSuccess;
    if (blk_elem && e == cudaSuccess) e = cudaMemcpy(blk_elem, P->blk_elem, sizeof(int32_t) * (P->n_blocks + 1), cudaMemcpyDeviceToHost);
    if (blk_occ && e == cudaSuccess) e = cudaMemcpy(blk_occ, P->blk_occ, sizeof(int32_t) * (P->n_blocks + 1), cudaMemcpyDeviceToHost);
    if (occ_node && e == cudaSuccess) e = cudaMemcpy(occ_node, P->occ_node, sizeof(int32_t) * P->n_occ, cudaMemcpyDeviceToHost);
    if (occ_ent_ptr && e == cudaSuccess) e = cudaMemcpy(occ_ent_ptr, P->occ_ent_ptr, sizeof(int32_t) * (P->n_occ + 1), cudaMemcpyDeviceToHost);
    if (loc_ent && e == cudaSuccess)
        e = cudaMemcpy(loc_ent, P->loc_ent, sizeof(uint16_t) * (size_t)P->n_elems * (P->dim + 1), cudaMemcpyDeviceToHost);
    if (elem_perm && e == cudaSuccess) {
        if (P->elem_perm) {
            e = cudaMemcpy(elem_perm, P->elem_perm, sizeof(int32_t) * (size_t)P->n_elems, cudaMemcpyDeviceToHost);
        } else {
            for (int32_t i = 0; i < P->n_elems; ++i) elem_perm[i] = i;
        }
    }
    if (e != cudaSuccess) return cuda_status(e, "pfem_plan_export");
    return PFEM_OK;
}

size_t pfem_workspace_bytes(const pfem_mesh* m, int32_t n_samples) {
    if (check_mesh(m, true) != PFEM_OK || n_samples <= 0) return 0;
    const Plan* P = reinterpret_cast<const Plan*>(m->plan);
    return ws_layout(*P, n_samples, m->dtype == PFEM_F64 ? 8 : 4).total;
}

pfem_status pfem_lame(int32_t dtype, int32_t kind, int64_t n, const void* p0, int64_t stride0, const void* p1,
                      int64_t stride1, void* mu, void* lam, void* stream) {
    if (!p0 || !p1 || !mu || !lam || n < 0 || kind < 0 || kind > 2) { set_error("pfem_lame: bad argument"); return PFEM_ERR_ARG; }
    if (n == 0) return PFEM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned g = (unsigned)((n + 255) / 256);
    if (dtype == PFEM_F32)
        k_lame<float><<<g, 256, 0, s>>>(n, kind, (const float*)p0, stride0, (const float*)p1, stride1, (float*)mu, (float*)lam);
    else if (dtype == PFEM_F64)
        k_lame<double><<<g, 256, 0, s>>>(n, kind, (const double*)p0, stride0, (const double*)p1, stride1, (double*)mu, (double*)lam);
    else { set_error("bad dtype"); return PFEM_ERR_ARG; }
    PFEM_LAUNCH_CHECK("k_lame");
    return PFEM_OK;
}

pfem_status pfem_energy(const pfem_mesh* m, const pfem_material* mat, int32_t n_samples, const void* u,
                        int64_t sample_stride, const void* f_ext, void* elem_energy, void* totals, void* residual,
                        int32_t mode, pfem_flags* flags, void* ws, size_t ws_bytes, void* stream) {
    pfem_status st = common_checks(m, mat, n_samples, sample_stride, mode, ws, ws_bytes);
    if (st) return st;
    if (!u || !totals) { set_error("pfem_energy: u and totals are required"); return PFEM_ERR_ARG; }
    Call c{};
    c.m = m;
    c.P = reinterpret_cast<const Plan*>(m->plan);
    c.op = residual ? OP_ENERGY_RESIDUAL : OP_ENERGY;
    c.model = mat->model;
    c.mode = mode;
    c.S = n_samples;
    c.sstride = sample_stride;
    c.mat = *mat;
    c.u = u;
    c.f_ext = f_ext;
    c.W_e = elem_energy;
    c.totals = totals;
    c.out = residual;
    c.flags = flags;
    c.ws = ws;
    c.ws_bytes = ws_bytes;
    c.stream = (cudaStream_t)stream;
    return run(c);
}

pfem_status pfem_pretrain_loss(const pfem_mesh* m, const pfem_material* mat, int32_t n_samples, const void* H,
                               int64_t sample_stride, const void* phi, const void* f_ext, void* u, void* totals,
                               void* grad, double* loss, int32_t mode, pfem_flags* flags, void* ws, size_t ws_bytes,
                               void* stream) {
    if (m && m->elem_type != PFEM_ELEM_SIMPLEX) { set_error("pfem_pretrain_loss: simplex meshes only"); return PFEM_ERR_ARG; }
    pfem_status st = common_checks(m, mat, n_samples, sample_stride, mode, ws, ws_bytes);
    if (st) return st;
    if (!H || !totals || !grad || !loss) { set_error("pfem_pretrain_loss: H, totals, grad and loss are required"); return PFEM_ERR_ARG; }
    if (phi && !u) { set_error("pfem_pretrain_loss: u (the ansatz field) is required with phi"); return PFEM_ERR_ARG; }
    cudaStream_t s = (cudaStream_t)stream;
    const void* uu = H;
    if (phi) {
        if ((st = run_pretrain_stage(m, n_samples, sample_stride, H, phi, u, 0, nullptr, nullptr, nullptr, nullptr, s)))
            return st;
        uu = u;
    }
    Call c{};
    c.m = m;
    c.P = reinterpret_cast<const Plan*>(m->plan);
    c.op = OP_ENERGY_RESIDUAL;
    c.model = mat->model;
    c.mode = mode;
    c.S = n_samples;
    c.sstride = sample_stride;
    c.mat = *mat;
    c.u = uu;
    c.f_ext = f_ext;
    c.totals = totals;
    c.out = grad;
    c.flags = flags;
    c.ws = ws;
    c.ws_bytes = ws_bytes;
    c.stream = s;
    // CSR: the epilogue is applied where kernels A / B write each DOF, and kernel B's last CTA
    // writes the loss; COLOUR (read-modify-write passes): a separate epilogue pass
    const bool fused = mode == PFEM_ASSEMBLE_CSR;
    c.ep = fused ? 1 : 0;
    c.ep_phi = phi;
    c.ep_loss = loss;
    if ((st = run(c))) return st;
    if (fused) return PFEM_OK;
    return run_pretrain_stage(m, n_samples, sample_stride, nullptr, phi, nullptr, 1, f_ext, grad, totals, loss, s);
}

size_t pfem_heat_workspace_bytes(const pfem_mesh* m, int32_t n_samples) {
    if (check_mesh(m, true) != PFEM_OK || n_samples <= 0) return 0;
    return heat_ws_bytes(m, n_samples);
}

pfem_status pfem_heat(const pfem_mesh* m, const void* k, int64_t k_stride, int32_t n_samples, const void* T,
                      int64_t sample_stride, const void* f_nodal, void* elem_energy, void* totals, void* flux,
                      int32_t options, void* ws, size_t ws_bytes, void* stream) {
    pfem_status st = check_mesh(m, true);   // runs on the prepared mesh (the flux path reads the plan)
    if (!st && m->elem_type != PFEM_ELEM_SIMPLEX) { set_error("pfem_heat: simplex meshes only"); return PFEM_ERR_ARG; }
    if (st) return st;
    if (!k || !T) { set_error("pfem_heat: k and T are required"); return PFEM_ERR_ARG; }
    if (k_stride < 0) { set_error("pfem_heat: negative k_stride"); return PFEM_ERR_ARG; }
    if (n_samples <= 0) { set_error("n_samples must be positive"); return PFEM_ERR_ARG; }
    if (sample_stride < m->n_nodes && n_samples > 1) { set_error("sample_stride smaller than n_nodes"); return PFEM_ERR_ARG; }
    if (totals && !elem_energy) { set_error("pfem_heat: totals need elem_energy"); return PFEM_ERR_ARG; }
    if ((totals && !ws) || (ws && ws_bytes < heat_ws_bytes(m, n_samples))) {
        set_error("pfem_heat: workspace too small (pfem_heat_workspace_bytes)");
        return PFEM_ERR_CAPACITY;
    }
    if (flux && (!m->csr_ptr || !m->csr_ent)) { set_error("pfem_heat: mesh CSR missing (prepare first)"); return PFEM_ERR_ARG; }
    if (options & ~PFEM_HEAT_GEOMETRY_ON_THE_FLY) { set_error("pfem_heat: unknown options"); return PFEM_ERR_ARG; }
    if ((options & PFEM_HEAT_GEOMETRY_ON_THE_FLY) && !m->coords) { set_error("pfem_heat: on-the-fly geometry needs coords"); return PFEM_ERR_ARG; }
    return run_heat(m, k, k_stride, n_samples, T, sample_stride, f_nodal, elem_energy, totals, flux, ws,
                    (options & PFEM_HEAT_GEOMETRY_ON_THE_FLY) ? 1 : 0, (cudaStream_t)stream);
}

pfem_status pfem_residual(const pfem_mesh* m, const pfem_material* mat, int32_t n_samples, const void* u,
                          int64_t sample_stride, void* residual, int32_t mode, pfem_flags* flags, void* ws,
                          size_t ws_bytes, void* stream) {
    pfem_status st = common_checks(m, mat, n_samples, sample_stride, mode, ws, ws_bytes);
    if (st) return st;
    if (!u || !residual) { set_error("pfem_residual: u and residual are required"); return PFEM_ERR_ARG; }
    Call c{};
    c.m = m;
    c.P = reinterpret_cast<const Plan*>(m->plan);
    c.op = OP_RESIDUAL;
    c.model = mat->model;
    c.mode = mode;
    c.S = n_samples;
    c.sstride = sample_stride;
    c.mat = *mat;
    c.u = u;
    c.out = residual;
    c.flags = flags;
    c.ws = ws;
    c.ws_bytes = ws_bytes;
    c.stream = (cudaStream_t)stream;
    return run(c);
}

pfem_status pfem_tangent_apply(const pfem_mesh* m, const pfem_material* mat, int32_t n_samples, const void* u,
                               const void* v, void* Kv, int64_t sample_stride, const uint8_t* dirichlet_mask,
                               int32_t mode, pfem_flags* flags, void* ws, size_t ws_bytes, void* stream) {
    pfem_status st = common_checks(m, mat, n_samples, sample_stride, mode, ws, ws_bytes);
    if (st) return st;
    if (!v || !Kv) { set_error("pfem_tangent_apply: v and Kv are required"); return PFEM_ERR_ARG; }
    if (mat->model == PFEM_NEOHOOKEAN && !u) { set_error("pfem_tangent_apply: Neo-Hookean needs u"); return PFEM_ERR_ARG; }
    Call c{};
    c.m = m;
    c.P = reinterpret_cast<const Plan*>(m->plan);
    c.op = OP_TANGENT;
    c.model = mat->model;
    c.mode = mode;
    c.S = n_samples;
    c.sstride = sample_stride;
    c.mat = *mat;
    c.u = u;
    c.v = v;
    c.mask = dirichlet_mask;
    c.out = Kv;
    c.flags = flags;
    c.ws = ws;
    c.ws_bytes = ws_bytes;
    c.stream = (cudaStream_t)stream;
    return run(c);
}

size_t pfem_cg_workspace_bytes(const pfem_mesh* m) {
    if (check_mesh(m, true) != PFEM_OK) return 0;
    return cg_ws_bytes(*reinterpret_cast<const Plan*>(m->plan), m->dtype);
}

pfem_status pfem_tangent_diag(const pfem_mesh* m, const pfem_material* mat, const void* u_state, void* diag,
                              const uint8_t* mask, void* stream) {
    pfem_status st = check_mesh(m, true);
    if (st) return st;
    if (m->elem_type != PFEM_ELEM_SIMPLEX) { set_error("pfem_tangent_diag: simplex meshes only"); return PFEM_ERR_ARG; }
    if ((st = check_mat(mat))) return st;
    if (!diag) { set_error("pfem_tangent_diag: diag is required"); return PFEM_ERR_ARG; }
    if (mat->model == PFEM_NEOHOOKEAN && !u_state) { set_error("pfem_tangent_diag: Neo-Hookean needs u_state"); return PFEM_ERR_ARG; }
    st = run_tangent_diag(m, mat, u_state, mask, 0, diag, (cudaStream_t)stream);
    if (st == PFEM_OK) count_launch();
    return st;
}

pfem_status pfem_pcg(const pfem_mesh* m, const pfem_material* mat, const void* u_state, const void* rhs,
                     const uint8_t* mask, int32_t precond, void* x, double tol, int32_t max_iter, int32_t mode,
                     double* history, pfem_cg_report* report, void* ws, size_t ws_bytes, void* stream) {
    if (precond != PFEM_PRECOND_NONE && precond != PFEM_PRECOND_JACOBI) { set_error("pfem_pcg: bad precond"); return PFEM_ERR_ARG; }
    if (precond == PFEM_PRECOND_JACOBI && m && m->elem_type != PFEM_ELEM_SIMPLEX) {
        set_error("pfem_pcg: Jacobi preconditioning on simplex meshes only");
        return PFEM_ERR_ARG;
    }
    pfem_status st = check_mesh(m, true);
    if (st) return st;
    if ((st = check_mat(mat))) return st;
    if (!rhs || !x || !report || !ws) { set_error("pfem_pcg: NULL argument"); return PFEM_ERR_ARG; }
    if (mat->model == PFEM_NEOHOOKEAN && !u_state) { set_error("pfem_pcg: Neo-Hookean needs u_state"); return PFEM_ERR_ARG; }
    if (!(tol >= 0.0) || max_iter < 0) { set_error("pfem_pcg: bad tol / max_iter"); return PFEM_ERR_ARG; }
    if (mode != PFEM_ASSEMBLE_CSR && mode != PFEM_ASSEMBLE_COLOUR) { set_error("bad assembly mode"); return PFEM_ERR_ARG; }
    if (ws_bytes < pfem_cg_workspace_bytes(m)) { set_error("pfem_pcg: workspace too small"); return PFEM_ERR_CAPACITY; }
    memset(report, 0, sizeof(*report));
    return run_cg(m, mat, u_state, rhs, mask, x, tol, max_iter, mode, history, report, ws, (cudaStream_t)stream,
                  precond);
}

pfem_status pfem_cg(const pfem_mesh* m, const pfem_material* mat, const void* u_state, const void* rhs,
                    const uint8_t* mask, void* x, double tol, int32_t max_iter, int32_t mode, double* history,
                    pfem_cg_report* report, void* ws, size_t ws_bytes, void* stream) {
    pfem_status st = check_mesh(m, true);
    if (st) return st;
    if ((st = check_mat(mat))) return st;
    if (!rhs || !x || !report || !ws) { set_error("pfem_cg: NULL argument"); return PFEM_ERR_ARG; }
    if (mat->model == PFEM_NEOHOOKEAN && !u_state) { set_error("pfem_cg: Neo-Hookean needs u_state"); return PFEM_ERR_ARG; }
    if (!(tol >= 0.0) || max_iter < 0) { set_error("pfem_cg: bad tol / max_iter"); return PFEM_ERR_ARG; }
    if (mode != PFEM_ASSEMBLE_CSR && mode != PFEM_ASSEMBLE_COLOUR) { set_error("bad assembly mode"); return PFEM_ERR_ARG; }
    if (ws_bytes < pfem_cg_workspace_bytes(m)) { set_error("pfem_cg: workspace too small"); return PFEM_ERR_CAPACITY; }
    memset(report, 0, sizeof(*report));
    return run_cg(m, mat, u_state, rhs, mask, x, tol, max_iter, mode, history, report, ws, (cudaStream_t)stream, 0);
}

size_t pfem_newton_workspace_bytes(const pfem_mesh* m) {
    if (check_mesh(m, true) != PFEM_OK) return 0;
    return newton_ws_bytes(*reinterpret_cast<const Plan*>(m->plan), m->dtype);
}

pfem_status pfem_newton(const pfem_mesh* m, const pfem_material* mat, void* u, const void* f_ext,
                        const uint8_t* mask, double tol, int32_t max_newton, double cg_tol, int32_t cg_max_iter,
                        int32_t mode, double* history, pfem_newton_report* report, void* ws, size_t ws_bytes,
                        void* stream) {
    pfem_status st = check_mesh(m, true);
    if (st) return st;
    if ((st = check_mat(mat))) return st;
    if (!u || !report || !ws) { set_error("pfem_newton: NULL argument"); return PFEM_ERR_ARG; }
    if (!(tol >= 0.0) || !(cg_tol >= 0.0) || max_newton < 0 || cg_max_iter < 0) {
        set_error("pfem_newton: bad tol / iteration limits");
        return PFEM_ERR_ARG;
    }
    if (mode != PFEM_ASSEMBLE_CSR && mode != PFEM_ASSEMBLE_COLOUR) { set_error("bad assembly mode"); return PFEM_ERR_ARG; }
    if (ws_bytes < pfem_newton_workspace_bytes(m)) { set_error("pfem_newton: workspace too small"); return PFEM_ERR_CAPACITY; }
    memset(report, 0, sizeof(*report));
    return run_newton(m, mat, u, f_ext, mask, tol, max_newton, cg_tol, cg_max_iter, mode, history, report, ws,
                      (cudaStream_t)stream);
}

}  // extern "C"

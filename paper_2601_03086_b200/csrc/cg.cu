// cg.cu — warm-started conjugate gradient on the GPU (§8 row a7; App. B P:1021-1036,
// warm start P:395-417, skip rule P:419-423).
//
// Hestenes-Stiefel CG on A = (I-M) K (I-M) + M with b = (I-M)(f - K x_D), x_D = M x0.
// Scalars (rho, alpha, beta, the convergence test, the iteration count, the history)
// live on the device; every dot product is a fixed-grid, fixed-order reduction (no float
// atomics).  One iteration = 3 kernels:
//   k_assemble<TANGENT> (q = A p, fused p.q -> alpha in its last block)
//   k_cg_update          (x += alpha p, r -= alpha q, rho' = r.r -> test, beta in last block)
//   k_cg_dir             (p = r + beta p)
// captured B at a time in a CUDA graph and replayed until the device flag says done;
// converged / broken-down iterations exit at their first instruction.
//
// Jacobi preconditioning (reading R27): z = D^-1 r with
// D = diag(A) from k_tangent_diag; rho = r.z drives alpha and beta, the stop test stays on
// ||r|| (R8).  z is never stored: k_cg_update forms r.z with r.r, k_cg_dir p = D^-1 r + beta p.
#include <algorithm>

#include "launch.cuh"

namespace pfem {

constexpr int VEC_NT = 256;

constexpr int VEC_U = 4;          // independent elements per thread and pass (loads in flight)
constexpr int VEC_MAX_GRID = 2048;

struct VecRed {
    int32_t counter;
    int32_t pad[63];
    double part[VEC_MAX_GRID];
    double part2[VEC_MAX_GRID];   // second reduction of the same pass (PCG r.z)
};

// grid-stride passes of VEC_U elements per thread: i0 + u * stride, u < VEC_U
#define VEC_PASSES(n)                                                                       \
    const int64_t vstride_ = (int64_t)gridDim.x * VEC_NT;                                   \
    for (int64_t i0 = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i0 < (n); i0 += VEC_U * vstride_)
#define VEC_IDX(u) (i0 + (int64_t)(u) * vstride_)

__device__ __forceinline__ bool vec_last_block(VecRed* vr, double v, double* s_red, int* s_flag) {
    const double t = cta_sum<VEC_NT>(v, s_red);
    if (threadIdx.x == 0) {
        vr->part[blockIdx.x] = t;
        __threadfence();
        *s_flag = (atomicAdd(&vr->counter, 1) == (int)gridDim.x - 1);
    }
    __syncthreads();
    return *s_flag;
}

// two sums in one pass: per-CTA partials of both, the last CTA returns true
__device__ __forceinline__ bool vec_last_block2(VecRed* vr, double v, double v2, double* s_red, int* s_flag) {
    const double t2 = cta_sum<VEC_NT>(v2, s_red);
    if (threadIdx.x == 0) vr->part2[blockIdx.x] = t2;
    return vec_last_block(vr, v, s_red, s_flag);   // (its leading barrier orders the reuse of s_red)
}

__device__ __forceinline__ double vec_final_part2(VecRed* vr, double* s_red) {
    __threadfence();   // after the arrival that made this CTA the last one (as vec_final)
    double v = 0.0;
    for (int i0 = threadIdx.x; i0 < (int)gridDim.x; i0 += 8 * VEC_NT) {
        double w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = i0 + u * VEC_NT < (int)gridDim.x ? ld_relaxed(vr->part2 + i0 + u * VEC_NT) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) v += w[u];
    }
    return cta_sum<VEC_NT>(v, s_red);
}

// fixed-order sum of the per-CTA partials (called by the last CTA, valid in thread 0)
__device__ __forceinline__ double vec_final(VecRed* vr, double* s_red) {
    __threadfence();
    double v = 0.0;
    for (int i0 = threadIdx.x; i0 < (int)gridDim.x; i0 += 8 * VEC_NT) {   // loads 8 at a time
        double w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = i0 + u * VEC_NT < (int)gridDim.x ? ld_relaxed(vr->part + i0 + u * VEC_NT) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) v += w[u];
    }
    const double t = cta_sum<VEC_NT>(v, s_red);
    if (threadIdx.x == 0) vr->counter = 0;
    return t;
}

template <class T>
__global__ void __launch_bounds__(VEC_NT)
k_cg_masked_copy(int64_t n, const uint8_t* __restrict__ mask, const T* __restrict__ x, T* __restrict__ xd) {
    for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT)
        xd[i] = (mask && mask[i]) ? x[i] : T(0);
}

// b = (I-M)(f - K x_D); bnorm2 = b.b
template <class T>
__global__ void __launch_bounds__(VEC_NT)
k_cg_rhs(int64_t n, const uint8_t* __restrict__ mask, const T* __restrict__ f, const T* __restrict__ kxd,
         T* __restrict__ b, CgState* cg, VecRed* vr) {
    __shared__ double s_red[VEC_NT / 32];
    __shared__ int s_flag;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT) {
        T v = (mask && mask[i]) ? T(0) : f[i] - kxd[i];
        b[i] = v;
        acc += (double)v * (double)v;
    }
    if (!vec_last_block(vr, acc, s_red, &s_flag)) return;
    const double t = vec_final(vr, s_red);
    if (threadIdx.x == 0) cg->bnorm2 = t;
}

// r = b - A x (free DOFs), p = z = D^-1 r (z = r without preconditioner), rho = r.z,
// rho_new = r.r; skip rule / zero rhs
template <class T>
__global__ void __launch_bounds__(VEC_NT)
k_cg_r0(int64_t n, const uint8_t* __restrict__ mask, const T* __restrict__ b, const T* __restrict__ ax,
        T* __restrict__ r, T* __restrict__ p, T* __restrict__ x, CgState* cg, VecRed* vr, double* history,
        const T* __restrict__ dinv) {
    __shared__ double s_red[VEC_NT / 32];
    __shared__ int s_flag;
    double acc = 0.0, accz = 0.0;
    const bool zero_rhs = cg->bnorm2 == 0.0;
    for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT) {
        const bool c = mask && mask[i];
        T v = c ? T(0) : b[i] - ax[i];
        r[i] = v;
        const T z = dinv ? dinv[i] * v : v;
        p[i] = z;
        if (zero_rhs && !c) x[i] = T(0);
        acc += (double)v * (double)v;
        accz += (double)v * (double)z;
    }
    if (!vec_last_block2(vr, acc, accz, s_red, &s_flag)) return;
    const double tz = vec_final_part2(vr, s_red);
    const double t = vec_final(vr, s_red);
    if (threadIdx.x == 0) {
        cg->rho = dinv ? tz : t;
        cg->rho_new = t;
        cg->k = 0;
        cg->beta = 0.0;   // the pipelined first iteration forms p = z + 0 p (= z, as k_cg_r0 wrote it)
        const double bn2 = cg->bnorm2;
        cg->pad0 = bn2 > 0 ? sqrt(t / bn2) : 0.0;   // rel_res0
        if (history) history[0] = cg->pad0;
        if (bn2 == 0.0) {
            cg->rho = 0.0;
            cg->status = 1;
            cg->done = 1;
        } else if (t < cg->tol2 * bn2) {   // ||r|| < tol ||b||  (strict)
            cg->status = 1;
            cg->done = 1;
        } else if (cg->max_iter <= 0) {
            cg->status = 3;
            cg->done = 1;
        }
    }
}

template <class T, bool PRE>
__global__ void __launch_bounds__(VEC_NT)
k_cg_update(int64_t n, T* __restrict__ x, T* __restrict__ r, const T* __restrict__ p, const T* __restrict__ q,
            CgState* cg, VecRed* vr, double* history, const T* __restrict__ dinv) {
    __shared__ double s_red[VEC_NT / 32];
    __shared__ int s_flag;
    if (ld_relaxed_i(&cg->done)) return;
    const T alpha = (T)cg->alpha;
    double acc = 0.0, accz = 0.0;
    VEC_PASSES(n) {
        T xv[VEC_U], pv[VEC_U], qv[VEC_U], rv[VEC_U], dv[VEC_U];
#pragma unroll
        for (int u = 0; u < VEC_U; ++u) {
            const int64_t i = VEC_IDX(u);
            if (i < n) {
                xv[u] = x[i]; pv[u] = p[i]; qv[u] = q[i]; rv[u] = r[i];
                if (PRE) dv[u] = dinv[i];
            }
        }
#pragma unroll
        for (int u = 0; u < VEC_U; ++u) {
            const int64_t i = VEC_IDX(u);
            if (i >= n) break;
            x[i] = fma(alpha, pv[u], xv[u]);
            const T v = fma(-alpha, qv[u], rv[u]);
            r[i] = v;
            acc += (double)v * (double)v;
            if (PRE) accz += (double)v * (double)(dv[u] * v);
        }
    }
    double t, tz;
    if (PRE) {
        if (!vec_last_block2(vr, acc, accz, s_red, &s_flag)) return;
        tz = vec_final_part2(vr, s_red);
        t = vec_final(vr, s_red);
    } else {
        if (!vec_last_block(vr, acc, s_red, &s_flag)) return;
        t = vec_final(vr, s_red);
        tz = t;
    }
    if (threadIdx.x == 0) {
        const int k = cg->k + 1;
        cg->k = k;
        cg->rho_new = t;
        const double bn2 = cg->bnorm2;
        if (history) history[k] = sqrt(t / bn2);
        cg->beta = tz / cg->rho;
        cg->rho = tz;
        if (t < cg->tol2 * bn2) {
            cg->status = 1;
            cg->done = 1;
        } else if (k >= cg->max_iter) {
            cg->status = 3;
            cg->done = 1;
        }
    }
}

template <class T, bool PRE>
__global__ void __launch_bounds__(VEC_NT)
k_cg_dir(int64_t n, const T* __restrict__ r, T* __restrict__ p, const CgState* cg, const T* __restrict__ dinv) {
    if (ld_relaxed_i(&cg->done)) return;
    const T beta = (T)cg->beta;
    VEC_PASSES(n) {
        T pv[VEC_U], rv[VEC_U], dv[VEC_U];
#pragma unroll
        for (int u = 0; u < VEC_U; ++u) {
            const int64_t i = VEC_IDX(u);
            if (i < n) {
                pv[u] = p[i]; rv[u] = r[i];
                if (PRE) dv[u] = dinv[i];
            }
        }
#pragma unroll
        for (int u = 0; u < VEC_U; ++u) {
            const int64_t i = VEC_IDX(u);
            if (i < n) p[i] = fma(beta, pv[u], PRE ? dv[u] * rv[u] : rv[u]);
        }
    }
}

// Jacobi diagonal of A = (I-M) K(u) (I-M) + M (reading R27), one thread
// per node over the mesh's node -> (element, slot) CSR in ascending (e, a) order (the CSR sum
// of R12): the diagonal of the element tangent block of vertex a is
//   K_(a,i),(a,i) = V [mu |g_a|^2 + c ((F^-T g_a)_i)^2],  c = lam + mu - lam ln J   (NH)
//   (linear: F^-T = I, c = lam + mu), from dP_ij/dF_kl of App. B P:1104-1115 with k = i.
// Constrained DOFs get 1.  invert: write 1/diag (1 where diag <= 0 or not finite).
template <int D, int MODEL, class T>
__global__ void __launch_bounds__(VEC_NT)
k_tangent_diag(int N, int E, const int32_t* __restrict__ csr_ptr, const int32_t* __restrict__ csr_ent,
               const int32_t* __restrict__ conn, const T* __restrict__ grad, const T* __restrict__ vol,
               MatArgs<T> mat, const T* __restrict__ u, const uint8_t* __restrict__ mask, int invert,
               T* __restrict__ out) {
    constexpr int NV = D + 1;
    for (int n = blockIdx.x * VEC_NT + threadIdx.x; n < N; n += gridDim.x * VEC_NT) {
        T acc[D];
#pragma unroll
        for (int i = 0; i < D; ++i) acc[i] = T(0);
        for (int k = __ldg(csr_ptr + n); k < __ldg(csr_ptr + n + 1); ++k) {
            const int ent = __ldg(csr_ent + k);
            const int e = ent / NV, a = ent - e * NV;
            Geo<D, T> G;
            load_geo<D, T>(e, E, conn, grad, vol, mat, G);   // mu, lam scaled by V_e
            T ga[D];   // grad N_a (grad N_0 = -sum of the others); compile-time register indices
#pragma unroll
            for (int j = 0; j < D; ++j) {
                T s = G.g[0][j];
#pragma unroll
                for (int b = 1; b < D; ++b) s += G.g[b][j];
                ga[j] = -s;
#pragma unroll
                for (int b = 0; b < D; ++b)
                    if (a == b + 1) ga[j] = G.g[b][j];
            }
            T gg = ga[0] * ga[0];
#pragma unroll
            for (int j = 1; j < D; ++j) gg = fma(ga[j], ga[j], gg);
            T Ag[D];
            T c;
            if constexpr (MODEL == MODEL_NH) {
                T x[NV][D], H[D][D];
                gather<D, T, T, false>(u, 0, nullptr, G, x);
                grad_of<D, T, T>(G, x, H);
                NhState<D, T> NS;
                nh_state<D, T>(H, NS);
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    T s = NS.A[i][0] * ga[0];
#pragma unroll
                    for (int j = 1; j < D; ++j) s = fma(NS.A[i][j], ga[j], s);
                    Ag[i] = s;
                }
                c = G.lam + G.mu - G.lam * NS.lnJ;
            } else {
#pragma unroll
                for (int i = 0; i < D; ++i) Ag[i] = ga[i];
                c = G.lam + G.mu;
            }
#pragma unroll
            for (int i = 0; i < D; ++i) acc[i] += fma(c * Ag[i], Ag[i], G.mu * gg);
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int64_t dof = (int64_t)n * D + i;
            T v = (mask && mask[dof]) ? T(1) : acc[i];
            if (invert) v = (v > T(0) && isfinite(v)) ? T(1) / v : T(1);
            out[dof] = v;
        }
    }
}

template <int D, class T>
pfem_status tangent_diag_impl(const pfem_mesh* m, const pfem_material* mat, const void* u, const uint8_t* mask,
                              int invert, void* out, cudaStream_t s) {
    MatArgs<T> ma;
    ma.kind = mat->kind;
    ma.p0 = (const T*)mat->p0;
    ma.p1 = (const T*)mat->p1;
    ma.s0 = mat->stride0;
    ma.s1 = mat->stride1;
    const int grid = std::max(1, std::min(65535, (m->n_nodes + VEC_NT - 1) / VEC_NT));
    if (mat->model == MODEL_NH)
        k_tangent_diag<D, MODEL_NH, T><<<grid, VEC_NT, 0, s>>>(m->n_nodes, m->n_elems, m->csr_ptr, m->csr_ent, m->conn,
                                                               (const T*)m->grad, (const T*)m->vol, ma, (const T*)u,
                                                               mask, invert, (T*)out);
    else
        k_tangent_diag<D, MODEL_LINEAR, T><<<grid, VEC_NT, 0, s>>>(m->n_nodes, m->n_elems, m->csr_ptr, m->csr_ent,
                                                                   m->conn, (const T*)m->grad, (const T*)m->vol, ma,
                                                                   (const T*)u, mask, invert, (T*)out);
    PFEM_LAUNCH_CHECK("k_tangent_diag");
    return PFEM_OK;
}

pfem_status run_tangent_diag(const pfem_mesh* m, const pfem_material* mat, const void* u, const uint8_t* mask,
                             int invert, void* out, cudaStream_t s) {
    if (m->dim == 2)
        return m->dtype == PFEM_F32 ? tangent_diag_impl<2, float>(m, mat, u, mask, invert, out, s)
                                    : tangent_diag_impl<2, double>(m, mat, u, mask, invert, out, s);
    return m->dtype == PFEM_F32 ? tangent_diag_impl<3, float>(m, mat, u, mask, invert, out, s)
                                : tangent_diag_impl<3, double>(m, mat, u, mask, invert, out, s);
}

// COLOUR-mode CG: p.q and alpha as a separate pass
template <class T>
__global__ void __launch_bounds__(VEC_NT)
k_cg_pq(int64_t n, const T* __restrict__ p, const T* __restrict__ q, CgState* cg, VecRed* vr) {
    __shared__ double s_red[VEC_NT / 32];
    __shared__ int s_flag;
    if (ld_relaxed_i(&cg->done)) return;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT)
        acc += (double)p[i] * (double)q[i];
    if (!vec_last_block(vr, acc, s_red, &s_flag)) return;
    const double t = vec_final(vr, s_red);
    if (threadIdx.x == 0) {
        cg->pq = t;
        if (!(t > 0.0)) {
            cg->status = 2;
            cg->done = 1;
        } else {
            cg->alpha = cg->rho / t;
        }
    }
}

// ||b - A x|| over free DOFs -> pq slot (true residual)
template <class T>
__global__ void __launch_bounds__(VEC_NT)
k_cg_true(int64_t n, const uint8_t* __restrict__ mask, const T* __restrict__ b, const T* __restrict__ ax,
          CgState* cg, VecRed* vr) {
    __shared__ double s_red[VEC_NT / 32];
    __shared__ int s_flag;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT) {
        if (mask && mask[i]) continue;
        const double d = (double)b[i] - (double)ax[i];
        acc += d * d;
    }
    if (!vec_last_block(vr, acc, s_red, &s_flag)) return;
    const double t = vec_final(vr, s_red);
    if (threadIdx.x == 0) cg->pq = t;
}

struct CgWs {
    size_t state, vr, r, p, p2, q, b, dinv, asmws, total;
};

inline CgWs cg_layout(const Plan& P, size_t tsize) {
    CgWs L;
    size_t o = 0;
    const size_t nvec = align_up(tsize * (size_t)P.n_nodes * P.dim, 256);
    L.state = o; o += align_up(sizeof(CgState), 256);
    L.vr = o;    o += align_up(sizeof(VecRed), 256);
    L.r = o;     o += nvec;
    L.p = o;     o += nvec;
    L.p2 = o;    o += nvec;   // second direction buffer of the pipelined (CSR-mode) iteration
    L.q = o;     o += nvec;
    L.b = o;     o += nvec;
    L.dinv = o;  o += nvec;
    L.asmws = o; o += ws_layout(P, 1, tsize).total;
    L.total = o;
    return L;
}

size_t cg_ws_bytes(const Plan& P, int dtype) {
    return cg_layout(P, dtype == PFEM_F64 ? 8 : 4).total;
}

template <int D, class T>
static pfem_status tangent(const pfem_mesh* m, const Plan* P, const pfem_material* mat, const void* u,
                           const void* v, void* out, const uint8_t* mask, int mode, void* asmws, CgState* cg,
                           cudaStream_t s, const void* fuse_r = nullptr, const void* fuse_pold = nullptr,
                           const void* fuse_dinv = nullptr) {
    Call c{};
    c.m = m;
    c.P = P;
    c.op = OP_TANGENT;
    c.model = mat->model;
    c.mode = mode;
    c.S = 1;
    c.sstride = (int64_t)P->n_nodes * D;
    c.mat = *mat;
    c.u = u;
    c.v = v;
    c.mask = mask;
    c.out = out;
    c.ws = asmws;
    c.stream = s;
    c.cg = mode == PFEM_ASSEMBLE_CSR ? cg : nullptr;
    c.cg_r = fuse_r;
    c.cg_pold = fuse_pold;
    c.cg_dinv = fuse_dinv;
    return run_assemble<D, T>(c);
}

// Instantiated CG graphs, reused across calls: a graph bakes in every pointer and launch
// parameter of its B captured iterations, so it is keyed on all of them (plan serial, mesh
// arrays, material, state, mask, solution, workspace, history, B, mode, preconditioner).
// A few per host thread; the least recently captured one is replaced.
struct CgGraphKey {
    uint64_t serial;
    const void* ptr[12];
    int64_t val[8];
    bool operator==(const CgGraphKey& o) const {
        if (serial != o.serial) return false;
        for (int i = 0; i < 12; ++i)
            if (ptr[i] != o.ptr[i]) return false;
        for (int i = 0; i < 8; ++i)
            if (val[i] != o.val[i]) return false;
        return true;
    }
};
struct CgGraphEntry {
    CgGraphKey key;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t per_graph = 0;
    int device = -1;
};
constexpr int CG_GRAPH_CACHE = 4;
static thread_local CgGraphEntry g_cg_graphs[CG_GRAPH_CACHE];
static thread_local int g_cg_next = 0;
static thread_local cudaStream_t g_cg_stream = nullptr;
static thread_local int g_cg_stream_dev = -1;

template <int D, class T>
pfem_status cg_impl(const pfem_mesh* m, const pfem_material* mat, const void* u_state, const void* rhs,
                    const uint8_t* mask, void* xv, double tol, int max_iter, int mode, double* history,
                    pfem_cg_report* rep, void* ws, cudaStream_t s, int precond = 0) {
    const Plan* P = reinterpret_cast<const Plan*>(m->plan);
    const CgWs L = cg_layout(*P, sizeof(T));
    char* w = (char*)ws;
    CgState* st = (CgState*)(w + L.state);
    VecRed* vr = (VecRed*)(w + L.vr);
    T* r = (T*)(w + L.r);
    T* p = (T*)(w + L.p);
    T* p2 = (T*)(w + L.p2);
    T* q = (T*)(w + L.q);
    T* b = (T*)(w + L.b);
    T* dinv = precond ? (T*)(w + L.dinv) : nullptr;
    T* x = (T*)xv;
    void* asmws = w + L.asmws;
    const int64_t n = (int64_t)P->n_nodes * D;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int G = std::min(VEC_MAX_GRID, 8 * nsm);   // fixed grid => fixed reduction order
    CgState h{};
    h.tol2 = tol * tol;
    h.max_iter = max_iter;
    PFEM_CUDA_TRY(cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    PFEM_CUDA_TRY(cudaMemsetAsync(vr, 0, sizeof(int32_t), s));
    // b = (I-M)(f - K x_D)
    k_cg_masked_copy<T><<<G, VEC_NT, 0, s>>>(n, mask, x, p);
    PFEM_LAUNCH_CHECK("k_cg_masked_copy");
    pfem_status e = tangent<D, T>(m, P, mat, u_state, p, q, nullptr, mode, asmws, nullptr, s);
    if (e != PFEM_OK) return e;
    k_cg_rhs<T><<<G, VEC_NT, 0, s>>>(n, mask, (const T*)rhs, q, b, st, vr);
    PFEM_LAUNCH_CHECK("k_cg_rhs");
    // Jacobi: D^-1 of the masked operator at u_state
    if (dinv) {
        e = tangent_diag_impl<D, T>(m, mat, u_state, mask, 1, dinv, s);
        if (e != PFEM_OK) return e;
        count_launch();
    }
    // r0 = b - A x0
    e = tangent<D, T>(m, P, mat, u_state, x, q, mask, mode, asmws, nullptr, s);
    if (e != PFEM_OK) return e;
    k_cg_r0<T><<<G, VEC_NT, 0, s>>>(n, mask, b, q, r, p, x, st, vr, history, dinv);
    PFEM_LAUNCH_CHECK("k_cg_r0");
    PFEM_CUDA_TRY(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
    PFEM_CUDA_TRY(cudaStreamSynchronize(s));
    if (!h.done) {
        // capture B iterations into a graph on a private stream, replay on `s`
        // an even B keeps the two direction buffers of the pipelined loop aligned across replays
        const int B = std::max(1, std::min(32, max_iter + (max_iter & 1)));
        CgGraphKey key{};
        key.serial = P->serial;
        const void* kp[12] = {m->conn, m->grad, m->vol, m->coords, mat->p0, mat->p1, u_state, mask, x, ws, history,
                              (const void*)s};
        for (int i = 0; i < 12; ++i) key.ptr[i] = kp[i];
        const int64_t kv[8] = {B, mode, precond, mat->model, mat->kind, mat->stride0, mat->stride1,
                               (int64_t)m->geometry * 16 + (int64_t)sizeof(T)};
        for (int i = 0; i < 8; ++i) key.val[i] = kv[i];
        CgGraphEntry* hit = nullptr;
        for (auto& en : g_cg_graphs)
            if (en.exec && en.device == dev && en.key == key) hit = &en;
        cudaError_t cerr = cudaSuccess;
        if (!hit) {
        if (g_cg_stream == nullptr || g_cg_stream_dev != dev) {
            PFEM_CUDA_TRY(cudaStreamCreateWithFlags(&g_cg_stream, cudaStreamNonBlocking));
            g_cg_stream_dev = dev;
        }
        cudaStream_t cs = g_cg_stream;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        int64_t launches_before = pfem_launch_count(0);
        pfem_status ce = PFEM_OK;
        cerr = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
        if (cerr != cudaSuccess) return cuda_status(cerr, "cudaStreamBeginCapture");
        // pipelined iteration (§8(f) row f3): the simplex CSR element kernel
        const bool fuse = mode == PFEM_ASSEMBLE_CSR && P->elem_type == PFEM_ELEM_SIMPLEX;
        for (int it = 0; it < B && ce == PFEM_OK; ++it) {
            if (fuse) {
                // K.v stages p_new = z + beta p_old from r and the other p buffer (its owners
                // store p_new), kernel B forms p.q and alpha; then x, r, r.r and beta: 3 launches
                T* pold = (it & 1) ? p2 : p;
                T* pnew = (it & 1) ? p : p2;
                ce = tangent<D, T>(m, P, mat, u_state, pnew, q, mask, mode, asmws, st, cs, r, pold, dinv);
                if (ce != PFEM_OK) break;
                if (dinv) k_cg_update<T, true><<<G, VEC_NT, 0, cs>>>(n, x, r, pnew, q, st, vr, history, dinv);
                else k_cg_update<T, false><<<G, VEC_NT, 0, cs>>>(n, x, r, pnew, q, st, vr, history, nullptr);
                count_launch();
                continue;
            }
            ce = tangent<D, T>(m, P, mat, u_state, p, q, mask, mode, asmws, st, cs);
            if (ce != PFEM_OK) break;
            if (!fuse) {   // (the simplex CSR kernel forms p.q and alpha itself)
                k_cg_pq<T><<<G, VEC_NT, 0, cs>>>(n, p, q, st, vr);
                count_launch();
            }
            if (dinv) {
                k_cg_update<T, true><<<G, VEC_NT, 0, cs>>>(n, x, r, p, q, st, vr, history, dinv);
                k_cg_dir<T, true><<<G, VEC_NT, 0, cs>>>(n, r, p, st, dinv);
            } else {
                k_cg_update<T, false><<<G, VEC_NT, 0, cs>>>(n, x, r, p, q, st, vr, history, nullptr);
                k_cg_dir<T, false><<<G, VEC_NT, 0, cs>>>(n, r, p, st, nullptr);
            }
            count_launch(2);
        }
        cerr = cudaStreamEndCapture(cs, &graph);
        const int64_t per_graph = pfem_launch_count(0) - launches_before;
        if (ce == PFEM_OK && cerr == cudaSuccess) cerr = cudaGraphInstantiate(&exec, graph, 0);
        if (ce != PFEM_OK || cerr != cudaSuccess) {
            if (graph) cudaGraphDestroy(graph);
            if (ce != PFEM_OK) return ce;
            return cuda_status(cerr, "cg graph capture");
        }
        // the captured launches were counted at capture; count replays instead
        count_launch((int)-per_graph);
        CgGraphEntry& en = g_cg_graphs[g_cg_next];
        g_cg_next = (g_cg_next + 1) % CG_GRAPH_CACHE;
        if (en.exec) {
            cudaGraphExecDestroy(en.exec);
            cudaGraphDestroy(en.graph);
        }
        en.key = key;
        en.graph = graph;
        en.exec = exec;
        en.per_graph = per_graph;
        en.device = dev;
        hit = &en;
        }
        cudaGraphExec_t exec = hit->exec;
        const int64_t per_graph = hit->per_graph;
        int launched = 0;
        while (true) {
            cerr = cudaGraphLaunch(exec, s);
            if (cerr != cudaSuccess) break;
            count_launch((int)per_graph);
            launched += B;
            cerr = cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s);
            if (cerr != cudaSuccess) break;
            cerr = cudaStreamSynchronize(s);
            if (cerr != cudaSuccess || h.done || launched >= max_iter + B) break;
        }
        if (cerr != cudaSuccess) return cuda_status(cerr, "cg loop");
    }
    // true residual ||b - A x|| / ||b||
    e = tangent<D, T>(m, P, mat, u_state, x, q, mask, mode, asmws, nullptr, s);
    if (e != PFEM_OK) return e;
    k_cg_true<T><<<G, VEC_NT, 0, s>>>(n, mask, b, q, st, vr);
    PFEM_LAUNCH_CHECK("k_cg_true");
    PFEM_CUDA_TRY(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
    PFEM_CUDA_TRY(cudaStreamSynchronize(s));
    rep->iterations = h.k;
    rep->status = h.status;
    rep->converged = h.status == 1;
    rep->bnorm = sqrt(h.bnorm2);
    rep->rel_res_final = h.bnorm2 > 0 ? sqrt(h.rho_new / h.bnorm2) : 0.0;
    rep->true_rel_res_final = h.bnorm2 > 0 ? sqrt(h.pq / h.bnorm2) : 0.0;
    rep->rel_res0 = h.pad0;
    if (h.status == 2) {
        set_error("CG breakdown: p.Ap <= 0");
        return PFEM_ERR_BREAKDOWN;
    }
    if (h.status != 1) {
        set_error("CG did not converge within max_iter");
        return PFEM_ERR_NOT_CONVERGED;
    }
    return PFEM_OK;
}

// ====================================================================================
// Newton-Raphson (App. B, warm start P:1141-1166; §8(f) row f1):
//   r(U_k) = f_int(U_k) - f_ext on free DOFs;  stop when ||r|| <= tol;
//   K(U_k) dU = -r by the masked CG above (dU = 0 on constrained DOFs, x0 = 0, relative
//   tolerance cg_tol; K^ext = 0: dead loads);  U_{k+1} = U_k + dU.
// One host sync per Newton step (the residual norm decides the loop).

// rhs = f_ext - f_int on free DOFs (0 on constrained), ||rhs||^2 -> *out
template <class T>
__global__ void __launch_bounds__(VEC_NT)
k_newton_rhs(int64_t n, const uint8_t* __restrict__ mask, const T* __restrict__ fext, const T* __restrict__ fint,
             T* __restrict__ rhs, VecRed* vr, double* out) {
    __shared__ double s_red[VEC_NT / 32];
    __shared__ int s_flag;
    double acc = 0.0;
    VEC_PASSES(n) {
        T fe[VEC_U], fi[VEC_U];
        uint8_t mk[VEC_U];
#pragma unroll
        for (int u = 0; u < VEC_U; ++u) {
            const int64_t i = VEC_IDX(u);
            if (i < n) {
                fe[u] = fext ? fext[i] : T(0);
                fi[u] = fint[i];
                mk[u] = mask ? mask[i] : 0;
            }
        }
#pragma unroll
        for (int u = 0; u < VEC_U; ++u) {
            const int64_t i = VEC_IDX(u);
            if (i >= n) break;
            const T v = mk[u] ? T(0) : fe[u] - fi[u];
            rhs[i] = v;
            acc += (double)v * (double)v;
        }
    }
    if (!vec_last_block(vr, acc, s_red, &s_flag)) return;
    const double t = vec_final(vr, s_red);
    if (threadIdx.x == 0) *out = t;
}

template <class T>
__global__ void __launch_bounds__(VEC_NT)
k_newton_add(int64_t n, const T* __restrict__ du, T* __restrict__ u) {
    VEC_PASSES(n) {
        T a[VEC_U], b[VEC_U];
#pragma unroll
        for (int k = 0; k < VEC_U; ++k) {
            const int64_t i = VEC_IDX(k);
            if (i < n) { a[k] = u[i]; b[k] = du[i]; }
        }
#pragma unroll
        for (int k = 0; k < VEC_U; ++k) {
            const int64_t i = VEC_IDX(k);
            if (i < n) u[i] = a[k] + b[k];
        }
    }
}

struct NewtonWs {
    size_t cg, fint, rhs, du, red, total;
};

inline NewtonWs newton_layout(const Plan& P, size_t tsize) {
    NewtonWs L;
    size_t o = 0;
    const size_t nvec = align_up(tsize * (size_t)P.n_nodes * P.dim, 256);
    L.cg = o;   o += align_up(cg_layout(P, tsize).total, 256);
    L.fint = o; o += nvec;
    L.rhs = o;  o += nvec;
    L.du = o;   o += nvec;
    L.red = o;  o += align_up(sizeof(VecRed) + 256, 256);
    L.total = o;
    return L;
}

size_t newton_ws_bytes(const Plan& P, int dtype) {
    return newton_layout(P, dtype == PFEM_F64 ? 8 : 4).total;
}

template <int D, class T>
pfem_status newton_impl(const pfem_mesh* m, const pfem_material* mat, void* uv, const void* fext,
                        const uint8_t* mask, double tol, int max_newton, double cg_tol, int cg_max_iter, int mode,
                        double* history, pfem_newton_report* rep, void* ws, cudaStream_t s) {
    const Plan* P = reinterpret_cast<const Plan*>(m->plan);
    const NewtonWs L = newton_layout(*P, sizeof(T));
    char* w = (char*)ws;
    void* cgws = w + L.cg;
    void* asmws = w + L.cg + cg_layout(*P, sizeof(T)).asmws;
    T* fint = (T*)(w + L.fint);
    T* rhs = (T*)(w + L.rhs);
    T* du = (T*)(w + L.du);
    VecRed* vr = (VecRed*)(w + L.red);
    double* nrm = (double*)(w + L.red + sizeof(VecRed));
    T* u = (T*)uv;
    const int64_t n = (int64_t)P->n_nodes * D;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int G = std::min(VEC_MAX_GRID, 8 * nsm);
    PFEM_CUDA_TRY(cudaMemsetAsync(vr, 0, sizeof(int32_t), s));
    for (int k = 0;; ++k) {
        // r = f_int(U_k) - f_ext (free DOFs)
        Call c{};
        c.m = m;
        c.P = P;
        c.op = OP_RESIDUAL;
        c.model = mat->model;
        c.mode = mode;
        c.S = 1;
        c.sstride = n;
        c.mat = *mat;
        c.u = u;
        c.out = fint;
        c.ws = asmws;
        c.stream = s;
        pfem_status e = run_assemble<D, T>(c);
        if (e != PFEM_OK) return e;
        k_newton_rhs<T><<<G, VEC_NT, 0, s>>>(n, mask, (const T*)fext, fint, rhs, vr, nrm);
        PFEM_LAUNCH_CHECK("k_newton_rhs");
        double r2 = 0.0;
        PFEM_CUDA_TRY(cudaMemcpyAsync(&r2, nrm, sizeof(double), cudaMemcpyDeviceToHost, s));
        PFEM_CUDA_TRY(cudaStreamSynchronize(s));
        const double rn = sqrt(r2);
        if (history) history[k] = rn;
        if (k == 0) rep->res0 = rn;
        rep->res_final = rn;
        rep->iterations = k;
        if (!(rn == rn)) {
            rep->status = 3;
            set_error("Newton: non-finite residual (inverted elements?)");
            return PFEM_ERR_NOT_CONVERGED;
        }
        if (rn <= tol) {
            rep->converged = 1;
            rep->status = 0;
            return PFEM_OK;
        }
        if (k >= max_newton) {
            rep->status = 1;
            set_error("Newton did not converge within max_newton");
            return PFEM_ERR_NOT_CONVERGED;
        }
        // K(U_k) dU = f_ext - f_int  (x0 = 0, so the constrained entries of dU stay 0)
        PFEM_CUDA_TRY(cudaMemsetAsync(du, 0, sizeof(T) * (size_t)n, s));
        pfem_cg_report crep{};
        e = cg_impl<D, T>(m, mat, u, rhs, mask, du, cg_tol, cg_max_iter, mode, nullptr, &crep, cgws, s);
        rep->cg_iterations += crep.iterations;
        if (e == PFEM_ERR_BREAKDOWN) {
            rep->status = 2;
            return e;
        }
        if (e != PFEM_OK && e != PFEM_ERR_NOT_CONVERGED) return e;   // an inexact step still progresses
        k_newton_add<T><<<G, VEC_NT, 0, s>>>(n, du, u);
        PFEM_LAUNCH_CHECK("k_newton_add");
    }
}

pfem_status run_newton(const pfem_mesh* m, const pfem_material* mat, void* u, const void* fext, const uint8_t* mask,
                       double tol, int max_newton, double cg_tol, int cg_max_iter, int mode, double* history,
                       pfem_newton_report* rep, void* ws, cudaStream_t s) {
    if (m->dim == 2)
        return m->dtype == PFEM_F32
                   ? newton_impl<2, float>(m, mat, u, fext, mask, tol, max_newton, cg_tol, cg_max_iter, mode, history, rep, ws, s)
                   : newton_impl<2, double>(m, mat, u, fext, mask, tol, max_newton, cg_tol, cg_max_iter, mode, history, rep, ws, s);
    return m->dtype == PFEM_F32
               ? newton_impl<3, float>(m, mat, u, fext, mask, tol, max_newton, cg_tol, cg_max_iter, mode, history, rep, ws, s)
               : newton_impl<3, double>(m, mat, u, fext, mask, tol, max_newton, cg_tol, cg_max_iter, mode, history, rep, ws, s);
}

pfem_status run_cg(const pfem_mesh* m, const pfem_material* mat, const void* u_state, const void* rhs,
                   const uint8_t* mask, void* x, double tol, int max_iter, int mode, double* history,
                   pfem_cg_report* rep, void* ws, cudaStream_t s, int precond) {
    if (m->dim == 2)
        return m->dtype == PFEM_F32 ? cg_impl<2, float>(m, mat, u_state, rhs, mask, x, tol, max_iter, mode, history, rep, ws, s, precond)
                                    : cg_impl<2, double>(m, mat, u_state, rhs, mask, x, tol, max_iter, mode, history, rep, ws, s, precond);
    return m->dtype == PFEM_F32 ? cg_impl<3, float>(m, mat, u_state, rhs, mask, x, tol, max_iter, mode, history, rep, ws, s, precond)
                                : cg_impl<3, double>(m, mat, u_state, rhs, mask, x, tol, max_iter, mode, history, rep, ws, s, precond);
}

}  // namespace pfem

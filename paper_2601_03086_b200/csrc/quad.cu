// quad.cu — Q4 / Q8 quadrilateral elements with Gauss quadrature: the
// paper's hyperelastic beam (50 x 50 linear quadrilaterals, §4.2) and Cook's membrane
// (30 x 30 Q8 serendipity).  2-D, plane strain, the constitutive laws and the
// cancellation-free arithmetic of the simplex kernels (element.cuh), integrated over each
// element by a tensor-product Gauss rule (2 x 2 for Q4, 3 x 3 for Q8):
//   prepare  k_quad_geometry: per element and quadrature point, in fp64 from the coordinates,
//            dN_a/dX = dN_a/dxi J^{-1} and w det J (isoparametric map X = N_a X_a, App. B
//            P:1060-1066), stored in the call dtype; det J <= 0 at any point is degenerate;
//            k_quad_entry_pos: the CSR entry of every (element, node)
//   energy / residual / tangent: k_quad_elem (thread per element and sample: W_e and the nodal
//            forces sum_q w det J P grad N_a, stored at their CSR entries), k_quad_node_sum
//            (thread per node and sample: its entries in CSR order, ascending (element, node) —
//            the CSR gather of reading R12), per-part totals by k_colour_totals (fixed order).
// No float atomics; every sum has a fixed order.
#include <algorithm>

#include "launch.cuh"

namespace pfem {

constexpr int QD_NT = 256;

template <int NV>
struct QuadTraits {
    static constexpr int NQ = NV == 4 ? 4 : 9;   // 2 x 2 / 3 x 3 Gauss points
    static constexpr int REC = 2 * NV + 1;       // dN/dX [NV][2], w det J
};

// shape-function derivatives w.r.t. (xi, eta) at a reference point (node order: corners
// counter-clockwise from (-1,-1), then the midsides of edges 01, 12, 23, 30)
template <int NV>
__device__ __forceinline__ void quad_dshape(double xi, double eta, double (&dN)[NV][2]) {
    const double cx[8] = {-1, 1, 1, -1, 0, 1, 0, -1};
    const double cy[8] = {-1, -1, 1, 1, -1, 0, 1, 0};
#pragma unroll
    for (int a = 0; a < (NV == 4 ? 4 : 4); ++a) {
        const double xa = cx[a], ya = cy[a];
        if constexpr (NV == 4) {
            dN[a][0] = 0.25 * xa * (1.0 + eta * ya);
            dN[a][1] = 0.25 * ya * (1.0 + xi * xa);
        } else {
            dN[a][0] = 0.25 * xa * (1.0 + eta * ya) * (2.0 * xi * xa + eta * ya);
            dN[a][1] = 0.25 * ya * (1.0 + xi * xa) * (xi * xa + 2.0 * eta * ya);
        }
    }
    if constexpr (NV == 8) {
#pragma unroll
        for (int a = 4; a < 8; ++a) {
            const double xa = cx[a], ya = cy[a];
            if (xa == 0.0) {
                dN[a][0] = -xi * (1.0 + eta * ya);
                dN[a][1] = 0.5 * ya * (1.0 - xi * xi);
            } else {
                dN[a][0] = 0.5 * xa * (1.0 - eta * eta);
                dN[a][1] = -eta * (1.0 + xi * xa);
            }
        }
    }
}

template <int NV>
__device__ __forceinline__ void gauss_point(int q, double& xi, double& eta, double& w) {
    if constexpr (NV == 4) {
        const double g = 0.57735026918962576451;   // 1/sqrt(3)
        xi = (q & 1) ? g : -g;
        eta = (q & 2) ? g : -g;
        w = 1.0;
    } else {
        const double g = 0.77459666924148337704;   // sqrt(3/5)
        const double pt[3] = {-g, 0.0, g}, wt[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
        const int i = q % 3, j = q / 3;
        xi = pt[i];
        eta = pt[j];
        w = wt[i] * wt[j];
    }
}

template <int NV, class T>
__global__ void __launch_bounds__(QD_NT)
k_quad_geometry(int E, const double* __restrict__ X, const int32_t* __restrict__ conn, T* __restrict__ geo,
                int* first_degenerate) {
    constexpr int NQ = QuadTraits<NV>::NQ, REC = QuadTraits<NV>::REC;
    const int e = blockIdx.x * QD_NT + threadIdx.x;
    if (e >= E) return;
    double x[NV][2];
#pragma unroll
    for (int a = 0; a < NV; ++a) {
        const int n = conn[(int64_t)e * NV + a];
        x[a][0] = X[(int64_t)n * 2];
        x[a][1] = X[(int64_t)n * 2 + 1];
    }
    T* out = geo + (int64_t)e * NQ * REC;
    for (int q = 0; q < NQ; ++q) {
        double xi, eta, w, dN[NV][2];
        gauss_point<NV>(q, xi, eta, w);
        quad_dshape<NV>(xi, eta, dN);
        double J[2][2] = {{0, 0}, {0, 0}};   // J_ij = sum_a X_{a,i} dN_a/dxi_j
#pragma unroll
        for (int a = 0; a < NV; ++a)
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) J[i][j] += x[a][i] * dN[a][j];
        const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        if (!(det > 0.0)) atomicMin(first_degenerate, e);
        const double r = 1.0 / det;
        const double Ji[2][2] = {{J[1][1] * r, -J[0][1] * r}, {-J[1][0] * r, J[0][0] * r}};
#pragma unroll
        for (int a = 0; a < NV; ++a)
#pragma unroll
            for (int k = 0; k < 2; ++k) out[q * REC + 2 * a + k] = (T)(dN[a][0] * Ji[0][k] + dN[a][1] * Ji[1][k]);
        out[q * REC + 2 * NV] = (T)(w * det);
    }
}

__global__ void k_quad_entry_pos(int64_t nnz, const int32_t* __restrict__ csr_ent, int32_t* __restrict__ pos) {
    const int64_t k = (int64_t)blockIdx.x * QD_NT + threadIdx.x;
    if (k < nnz) pos[csr_ent[k]] = (int32_t)k;
}

template <class T>
struct QuadArgs {
    int E, N, S;
    int64_t sstride;
    const int32_t* conn;
    const T* geo;
    const int32_t* pos;
    MatArgs<T> mat;
    const T* u;            // field (energy / residual) or NH state (tangent)
    const T* v;            // tangent direction
    const uint8_t* mask;
    T* W;                  // [S][E] element energies (W_e or workspace)
    T* ebuf;               // [S][nnz][2] nodal forces at their CSR entries
    Counters* ctr;
};

template <int NV, int MODEL, class T, int OP, bool MASKED>
__global__ void __launch_bounds__(QD_NT)
k_quad_elem(const QuadArgs<T> p) {
    constexpr int NQ = QuadTraits<NV>::NQ, REC = QuadTraits<NV>::REC;
    constexpr bool HAS_PSI = OP == OP_ENERGY || OP == OP_ENERGY_RESIDUAL;
    constexpr bool HAS_FORCE = OP != OP_ENERGY;
    const int64_t idx = (int64_t)blockIdx.x * QD_NT + threadIdx.x;
    if (idx >= (int64_t)p.E * p.S) return;
    const int s = (int)(idx / p.E), e = (int)(idx - (int64_t)s * p.E);
    int c[NV];
#pragma unroll
    for (int a = 0; a < NV; ++a) c[a] = __ldg(p.conn + (int64_t)e * NV + a);
    T mu, lam;
    lame_of<T>(p.mat.kind, __ldg(p.mat.p0 + (int64_t)e * p.mat.s0), __ldg(p.mat.p1 + (int64_t)e * p.mat.s1), mu, lam);
    const T* fld = (OP == OP_TANGENT ? p.v : p.u) + (int64_t)s * p.sstride;
    T x[NV][2], xu[NV][2];
#pragma unroll
    for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int64_t dof = (int64_t)c[a] * 2 + i;
            x[a][i] = (MASKED && __ldg(p.mask + dof)) ? T(0) : __ldg(fld + dof);
            if (OP == OP_TANGENT && MODEL == MODEL_NH) xu[a][i] = __ldg(p.u + (int64_t)s * p.sstride + dof);
        }
    T W = T(0), f[NV][2];
#pragma unroll
    for (int a = 0; a < NV; ++a) f[a][0] = f[a][1] = T(0);
    int bad = 0;
    const T* ge = p.geo + (int64_t)e * NQ * REC;
    for (int q = 0; q < NQ; ++q) {
        T g[NV][2];
#pragma unroll
        for (int a = 0; a < NV; ++a) {
            g[a][0] = __ldg(ge + q * REC + 2 * a);
            g[a][1] = __ldg(ge + q * REC + 2 * a + 1);
        }
        const T wd = __ldg(ge + q * REC + 2 * NV);
        Geo<2, T> G;   // (only the moduli are read by the constitutive functions)
        G.mu = wd * mu;
        G.lam = wd * lam;
        T H[2][2], P[2][2], psi = T(0);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                T h = x[0][i] * g[0][j];
#pragma unroll
                for (int a = 1; a < NV; ++a) h = fma(x[a][i], g[a][j], h);
                H[i][j] = h;
            }
        if constexpr (OP == OP_TANGENT) {
            NhState<2, T> NS;
            if constexpr (MODEL == MODEL_NH) {
                T Hu[2][2];
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        T h = xu[0][i] * g[0][j];
#pragma unroll
                        for (int a = 1; a < NV; ++a) h = fma(xu[a][i], g[a][j], h);
                        Hu[i][j] = h;
                    }
                nh_state<2, T>(Hu, NS);
                bad += n_bad(NS.x);
            }
            dstress<2, MODEL, T, T>(G, NS, H, P);
        } else {
            int b = 0;
            stress<2, MODEL, T, T, HAS_PSI>(G, H, P, psi, b);
            bad += b;
        }
        if (HAS_PSI) W += psi;
        if (HAS_FORCE) {
#pragma unroll
            for (int a = 0; a < NV; ++a)
#pragma unroll
                for (int i = 0; i < 2; ++i) f[a][i] += fma(P[i][0], g[a][0], P[i][1] * g[a][1]);
        }
    }
    if (MODEL == MODEL_NH && bad) {
        atomicAdd(&p.ctr->n_inv, 1);
        atomicMax(&p.ctr->first_inv, INT32_MAX - e);
    }
    if (HAS_PSI) {
        if (!isfinite(W)) atomicAdd(&p.ctr->n_nonfinite, 1);
        p.W[(int64_t)s * p.E + e] = W;
    }
    if (HAS_FORCE) {
        const int64_t nnz = (int64_t)p.E * NV;
#pragma unroll
        for (int a = 0; a < NV; ++a) {
            const int32_t pk = __ldg(p.pos + (int64_t)e * NV + a);
            PFEM_DCHECK(pk >= 0 && pk < nnz);
            const int64_t k = (int64_t)s * nnz + pk;
            p.ebuf[2 * k] = f[a][0];
            p.ebuf[2 * k + 1] = f[a][1];
        }
    }
}

// node sums in CSR order (ascending (element, node)); masked rows of the tangent: out = v
template <class T, bool MASKED>
__global__ void __launch_bounds__(QD_NT)
k_quad_node_sum(int N, int S, int64_t nnz, int64_t sstride, const int32_t* __restrict__ csr_ptr,
                const T* __restrict__ ebuf, const uint8_t* __restrict__ mask, const T* __restrict__ v,
                T* __restrict__ out) {
    const int64_t idx = (int64_t)blockIdx.x * QD_NT + threadIdx.x;
    if (idx >= (int64_t)N * S) return;
    const int s = (int)(idx / N), n = (int)(idx - (int64_t)s * N);
    T a0 = T(0), a1 = T(0);
    const T* eb = ebuf + (int64_t)s * nnz * 2;
    for (int k = __ldg(csr_ptr + n); k < __ldg(csr_ptr + n + 1); ++k) {
        a0 += eb[2 * (int64_t)k];
        a1 += eb[2 * (int64_t)k + 1];
    }
    const int64_t o = (int64_t)s * sstride + (int64_t)n * 2;
    if (MASKED) {
        if (__ldg(mask + (int64_t)n * 2)) a0 = __ldg(v + o);
        if (__ldg(mask + (int64_t)n * 2 + 1)) a1 = __ldg(v + o + 1);
    }
    out[o] = a0;
    out[o + 1] = a1;
}

size_t quad_ebuf_bytes(const Plan& P, int S, size_t tsize) {
    return tsize * (size_t)S * P.n_elems * P.nv * 2;
}

template <int NV, int MODEL, class T, int OP, bool MASKED>
static pfem_status quad_launch(const Call& c) {
    constexpr bool HAS_PSI = OP == OP_ENERGY || OP == OP_ENERGY_RESIDUAL;
    constexpr bool HAS_FORCE = OP != OP_ENERGY;
    const Plan& P = *c.P;
    cudaStream_t s = c.stream;
    AsmParams<T> ap = make_params<T>(c);   // counters, totals, f_ext, flags for k_colour_totals
    const WsLayout L = ws_layout(P, c.S, sizeof(T));
    char* w = (char*)c.ws;
    QuadArgs<T> q;
    q.E = P.n_elems;
    q.N = P.n_nodes;
    q.S = c.S;
    q.sstride = c.sstride;
    q.conn = c.m->conn;
    q.geo = (const T*)P.quad_geo;
    q.pos = P.quad_pos;
    q.mat.kind = c.mat.kind;
    q.mat.p0 = (const T*)c.mat.p0;
    q.mat.p1 = (const T*)c.mat.p1;
    q.mat.s0 = c.mat.stride0;
    q.mat.s1 = c.mat.stride1;
    q.u = (const T*)c.u;
    q.v = (const T*)c.v;
    q.mask = c.mask;
    q.W = c.W_e ? (T*)c.W_e : (T*)(w + L.wtmp);
    q.ebuf = (T*)(w + L.partial);
    q.ctr = (Counters*)(w + L.counters);
    const int64_t ne = (int64_t)P.n_elems * c.S;
    k_quad_elem<NV, MODEL, T, OP, MASKED><<<(unsigned)((ne + QD_NT - 1) / QD_NT), QD_NT, 0, s>>>(q);
    PFEM_LAUNCH_CHECK("k_quad_elem");
    if (HAS_FORCE) {
        const int64_t nn = (int64_t)P.n_nodes * c.S;
        k_quad_node_sum<T, MASKED><<<(unsigned)((nn + QD_NT - 1) / QD_NT), QD_NT, 0, s>>>(
            P.n_nodes, c.S, (int64_t)P.n_elems * NV, c.sstride, c.m->csr_ptr, q.ebuf, c.mask, (const T*)c.v, (T*)c.out);
        PFEM_LAUNCH_CHECK("k_quad_node_sum");
    }
    const int want = HAS_PSI && c.totals ? 1 : 0;
    k_colour_totals<2, T><<<want ? c.S * P.n_parts : 1, ASM_NT, 0, s>>>(ap, P.part_elem, P.part_node, q.W, want);
    PFEM_LAUNCH_CHECK("k_colour_totals");
    return PFEM_OK;
}

template <int NV, int MODEL, class T>
static pfem_status quad_op(const Call& c) {
    switch (c.op) {
        case OP_ENERGY: return quad_launch<NV, MODEL, T, OP_ENERGY, false>(c);
        case OP_ENERGY_RESIDUAL: return quad_launch<NV, MODEL, T, OP_ENERGY_RESIDUAL, false>(c);
        case OP_RESIDUAL: return quad_launch<NV, MODEL, T, OP_RESIDUAL, false>(c);
        case OP_TANGENT:
            return c.mask ? quad_launch<NV, MODEL, T, OP_TANGENT, true>(c) : quad_launch<NV, MODEL, T, OP_TANGENT, false>(c);
    }
    set_error("bad op");
    return PFEM_ERR_ARG;
}

template <class T>
pfem_status run_quad(const Call& c) {
    if (c.mode != PFEM_ASSEMBLE_CSR) {
        set_error("quadrilateral meshes assemble in CSR mode only");
        return PFEM_ERR_ARG;
    }
    const bool nh = c.model == MODEL_NH;
    if (c.P->nv == 4) return nh ? quad_op<4, MODEL_NH, T>(c) : quad_op<4, MODEL_LINEAR, T>(c);
    return nh ? quad_op<8, MODEL_NH, T>(c) : quad_op<8, MODEL_LINEAR, T>(c);
}
template pfem_status run_quad<float>(const Call&);
template pfem_status run_quad<double>(const Call&);

// prepare: quadrature-point geometry (degenerate if det J <= 0 anywhere) and entry positions
pfem_status quad_prepare_geometry(const pfem_mesh* m, Plan* P, cudaStream_t s) {
    const int E = m->n_elems, nv = P->nv, nq = nv == 4 ? 4 : 9, rec = 2 * nv + 1;
    const size_t ts = m->dtype == PFEM_F64 ? 8 : 4;
    const size_t gbytes = align_up(ts * (size_t)E * nq * rec, 256);
    const size_t pbytes = align_up(sizeof(int32_t) * (size_t)E * nv, 256);
    void* pool = nullptr;
    PFEM_CUDA_TRY(cudaMallocAsync(&pool, gbytes + pbytes + 256, s));
    P->pool_quad = pool;
    P->quad_geo = pool;
    P->quad_pos = (int32_t*)((char*)pool + gbytes);
    int* bad = (int*)((char*)pool + gbytes + pbytes);
    const int init = INT32_MAX;
    PFEM_CUDA_TRY(cudaMemcpyAsync(bad, &init, sizeof(int), cudaMemcpyHostToDevice, s));
    const unsigned g = (unsigned)((E + QD_NT - 1) / QD_NT);
    if (nv == 4) {
        if (ts == 4) k_quad_geometry<4, float><<<g, QD_NT, 0, s>>>(E, m->coords, m->conn, (float*)P->quad_geo, bad);
        else k_quad_geometry<4, double><<<g, QD_NT, 0, s>>>(E, m->coords, m->conn, (double*)P->quad_geo, bad);
    } else {
        if (ts == 4) k_quad_geometry<8, float><<<g, QD_NT, 0, s>>>(E, m->coords, m->conn, (float*)P->quad_geo, bad);
        else k_quad_geometry<8, double><<<g, QD_NT, 0, s>>>(E, m->coords, m->conn, (double*)P->quad_geo, bad);
    }
    PFEM_LAUNCH_CHECK("k_quad_geometry");
    const int64_t nnz = (int64_t)E * nv;
    k_quad_entry_pos<<<(unsigned)((nnz + QD_NT - 1) / QD_NT), QD_NT, 0, s>>>(nnz, m->csr_ent, P->quad_pos);
    PFEM_LAUNCH_CHECK("k_quad_entry_pos");
    int h = 0;
    PFEM_CUDA_TRY(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    PFEM_CUDA_TRY(cudaStreamSynchronize(s));
    if (h != INT32_MAX) {
        set_error("degenerate quadrilateral (det J <= 0 at a Gauss point)", h);
        return PFEM_ERR_DEGENERATE;
    }
    return PFEM_OK;
}

}  // namespace pfem

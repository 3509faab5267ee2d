// heat.cu — steady heat conduction, the paper's scalar example (Eq.
// poisson_equation P:186-198 and its energy form P:249-284), on the same P1 geometry and CSR:
//   grad T_e = sum_{a>=1} (T_a - T_0) grad N_a
//   W_e = 1/2 k_e V_e |grad T_e|^2
//   totals[s][k] = sum_{e in part k} W_e - sum_{n in part k} f_n T_n
//   r_n = sum_{(e,a): v_a(e) = n} k_e V_e grad T_e . grad N_a    (the tangent is r(v): linear)
// One DOF per node.  Energies: thread per element; totals: one CTA per (sample, part), fixed
// order; fluxes: thread per node over its CSR row in ascending (e, a) order, each entry
// re-forming its element's gradient from the gathered nodal values (the per-element work is a
// few FMAs, so the recomputation is cheaper than a force buffer).  No float atomics.
#include "launch.cuh"

namespace pfem {

constexpr int HT_NT = 256;

template <int D, class T>
__device__ __forceinline__ void heat_grad(const int32_t* __restrict__ conn, const T* __restrict__ grad, int E,
                                          int e, const T* __restrict__ Ts, T g[D][D], T gT[D]) {
    constexpr int NV = D + 1;
    int c[NV];
#pragma unroll
    for (int a = 0; a < NV; ++a) c[a] = __ldg(conn + (int64_t)e * NV + a);
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int j = 0; j < D; ++j) g[a][j] = __ldg(grad + (int64_t)(a * D + j) * E + e);
    const T t0 = __ldg(Ts + c[0]);
    T dt[D];
#pragma unroll
    for (int a = 0; a < D; ++a) dt[a] = __ldg(Ts + c[a + 1]) - t0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        T s = dt[0] * g[0][j];
#pragma unroll
        for (int a = 1; a < D; ++a) s = fma(dt[a], g[a][j], s);
        gT[j] = s;
    }
}

template <int D, class T>
__global__ void __launch_bounds__(HT_NT)
k_heat_elem(int E, int N, int S, int64_t sstride, const int32_t* __restrict__ conn, const T* __restrict__ grad,
            const T* __restrict__ vol, const T* __restrict__ k, int64_t kstride, const T* __restrict__ Tf,
            T* __restrict__ W) {
    for (int e = blockIdx.x * HT_NT + threadIdx.x; e < E; e += gridDim.x * HT_NT) {
        const T hv = T(0.5) * __ldg(k + (int64_t)e * kstride) * __ldg(vol + e);
        for (int s = 0; s < S; ++s) {
            T g[D][D], gT[D];
            heat_grad<D, T>(conn, grad, E, e, Tf + (int64_t)s * sstride, g, gT);
            T gg = gT[0] * gT[0];
#pragma unroll
            for (int j = 1; j < D; ++j) gg = fma(gT[j], gT[j], gg);
            W[(int64_t)s * E + e] = hv * gg;
        }
    }
}

constexpr int HT_SLICES = 64;   // fixed slices per (sample, part): a fixed summation order

// stage 1, CTA (slice g, part k, sample s): the part's elements and nodes cut into HT_SLICES
// equal slices; partial[s][k][g] = sum of the slice's W_e - f.T over the slice's nodes
template <class T>
__global__ void __launch_bounds__(HT_NT)
k_heat_partials(int E, int N, int K, int64_t sstride, const int32_t* __restrict__ part_elem,
                const int32_t* __restrict__ part_node, const T* __restrict__ W, const T* __restrict__ f,
                const T* __restrict__ Tf, double* __restrict__ partial) {
    __shared__ double s_red[HT_NT / 32];
    const int g = blockIdx.x, kp = blockIdx.y, s = blockIdx.z;
    const int e0 = part_elem ? part_elem[kp] : 0, e1 = part_elem ? part_elem[kp + 1] : E;
    const int ce = (e1 - e0 + HT_SLICES - 1) / HT_SLICES;
    const int a0 = min(e1, e0 + g * ce), a1 = min(e1, a0 + ce);
    double acc = 0.0;
    for (int e = a0 + threadIdx.x; e < a1; e += HT_NT) acc += (double)W[(int64_t)s * E + e];
    if (f) {
        const int n0 = part_node ? part_node[kp] : 0, n1 = part_node ? part_node[kp + 1] : N;
        const int cn = (n1 - n0 + HT_SLICES - 1) / HT_SLICES;
        const int b0 = min(n1, n0 + g * cn), b1 = min(n1, b0 + cn);
        for (int n = b0 + threadIdx.x; n < b1; n += HT_NT) acc -= (double)f[n] * (double)Tf[(int64_t)s * sstride + n];
    }
    const double t = cta_sum<HT_NT>(acc, s_red);
    if (threadIdx.x == 0) partial[((int64_t)s * K + kp) * HT_SLICES + g] = t;
}

// stage 2: totals[s][k] = sum of the part's slice partials in slice order
template <class T>
__global__ void __launch_bounds__(HT_NT)
k_heat_totals(int SK, const double* __restrict__ partial, T* __restrict__ totals) {
    const int i = blockIdx.x * HT_NT + threadIdx.x;
    if (i >= SK) return;
    double t = 0.0;
    for (int g = 0; g < HT_SLICES; ++g) t += partial[(int64_t)i * HT_SLICES + g];
    totals[i] = (T)t;
}

// fluxes: thread per node, entries in CSR order; the entry's geometry is loaded once for up to
// HT_SC samples (each sample's sum still runs over the entries in ascending order)
constexpr int HT_SC = 4;

template <int D, class T>
__global__ void __launch_bounds__(HT_NT)
k_heat_flux(int N, int E, int S, int64_t sstride, const int32_t* __restrict__ csr_ptr, const int32_t* __restrict__ csr_ent,
            const int32_t* __restrict__ conn, const T* __restrict__ grad, const T* __restrict__ vol,
            const T* __restrict__ k, int64_t kstride, const T* __restrict__ Tf, T* __restrict__ r) {
    constexpr int NV = D + 1;
    for (int n = blockIdx.x * HT_NT + threadIdx.x; n < N; n += gridDim.x * HT_NT) {
        const int k0 = __ldg(csr_ptr + n), k1 = __ldg(csr_ptr + n + 1);
        for (int s0 = 0; s0 < S; s0 += HT_SC) {
            const int nq = min(HT_SC, S - s0);
            T acc[HT_SC];
#pragma unroll
            for (int q = 0; q < HT_SC; ++q) acc[q] = T(0);
            for (int q = k0; q < k1; ++q) {
                const int ent = __ldg(csr_ent + q);
                const int e = ent / NV, a = ent - e * NV;
                int c[NV];
#pragma unroll
                for (int b = 0; b < NV; ++b) c[b] = __ldg(conn + (int64_t)e * NV + b);
                T g[D][D];
#pragma unroll
                for (int b = 0; b < D; ++b)
#pragma unroll
                    for (int j = 0; j < D; ++j) g[b][j] = __ldg(grad + (int64_t)(b * D + j) * E + e);
                T ga[D];   // grad N_a, grad N_0 = -sum (compile-time register indices)
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    T sm = g[0][j];
#pragma unroll
                    for (int b = 1; b < D; ++b) sm += g[b][j];
                    ga[j] = -sm;
#pragma unroll
                    for (int b = 0; b < D; ++b)
                        if (a == b + 1) ga[j] = g[b][j];
                }
                const T kv = __ldg(k + (int64_t)e * kstride) * __ldg(vol + e);
#pragma unroll
                for (int sq = 0; sq < HT_SC; ++sq) {
                    if (sq >= nq) break;
                    const T* Ts = Tf + (int64_t)(s0 + sq) * sstride;
                    const T t0 = __ldg(Ts + c[0]);
                    T dt[D];
#pragma unroll
                    for (int b = 0; b < D; ++b) dt[b] = __ldg(Ts + c[b + 1]) - t0;
                    T dg = T(0);
#pragma unroll
                    for (int j = 0; j < D; ++j) {
                        T gTj = dt[0] * g[0][j];
#pragma unroll
                        for (int b = 1; b < D; ++b) gTj = fma(dt[b], g[b][j], gTj);
                        dg = j == 0 ? gTj * ga[0] : fma(gTj, ga[j], dg);
                    }
                    acc[sq] = fma(kv, dg, acc[sq]);
                }
            }
#pragma unroll
            for (int sq = 0; sq < HT_SC; ++sq)
                if (sq < nq) r[(int64_t)(s0 + sq) * sstride + n] = acc[sq];
        }
    }
}

size_t heat_ec_bytes(const pfem_mesh* m);
// workspace: [ stamp | pos | entry buffer ] at offset 0 (their offsets depend only on the mesh,
// so one workspace may serve calls with different sample counts) | slice partials [S][K][slices]
size_t heat_ws_bytes(const pfem_mesh* m, int S) {
    return heat_ec_bytes(m) + ((sizeof(double) * (size_t)S * m->n_parts * HT_SLICES + 255) / 256 * 256);
}

// element-centric flux path (HT_EC): entry position of every (element, vertex) in the CSR,
// then per element the d+1 vertex fluxes of up to HT_SC samples stored at their CSR entries,
// then each node sums its contiguous entries in CSR order (the same order as k_heat_flux)
__global__ void __launch_bounds__(HT_NT)
k_heat_entry_pos(int64_t nnz, const int32_t* __restrict__ csr_ent, int32_t* __restrict__ pos,
                 const unsigned long long* __restrict__ stamp, unsigned long long key) {
    if (stamp[0] == key) return;   // this workspace already holds the positions of this plan
    const int64_t stride = (int64_t)gridDim.x * HT_NT;
    for (int64_t q = (int64_t)blockIdx.x * HT_NT + threadIdx.x; q < nnz; q += stride) pos[csr_ent[q]] = (int32_t)q;
}

// on-the-fly geometry (SURVEY §8(f) row f4 variant): grad N_a (rows of J^-1, J = [X_1 - X_0 | ..])
// and V = |det J| / d! formed in fp64 from the vertex coordinates (App. B), instead
// of reading the prepared gradients and volumes: fewer bytes per element, more arithmetic
template <int D, class T>
__device__ __forceinline__ void geometry_of(const double* __restrict__ X, const int (&c)[D + 1], T g[D][D], T& V) {
    double J[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int a = 0; a < D; ++a) J[i][a] = __ldg(X + (int64_t)c[a + 1] * D + i) - __ldg(X + (int64_t)c[0] * D + i);
    if constexpr (D == 2) {
        const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0], r = 1.0 / det;
        g[0][0] = (T)(J[1][1] * r);  g[0][1] = (T)(-J[0][1] * r);
        g[1][0] = (T)(-J[1][0] * r); g[1][1] = (T)(J[0][0] * r);
        V = (T)(fabs(det) * 0.5);
    } else {
        double cof[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
                cof[i][j] = J[i1][j1] * J[i2][j2] - J[i1][j2] * J[i2][j1];
            }
        const double det = J[0][0] * cof[0][0] + J[0][1] * cof[0][1] + J[0][2] * cof[0][2], r = 1.0 / det;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int j = 0; j < 3; ++j) g[a][j] = (T)(cof[j][a] * r);   // (J^-1)[a][j] = cof[j][a] / det
        V = (T)(fabs(det) / 6.0);
    }
}

template <int D, class T, bool OTF>
__global__ void __launch_bounds__(HT_NT)
k_heat_elem_flux(int E, int S, int s0, int64_t sstride, const int32_t* __restrict__ conn, const T* __restrict__ grad,
                 const T* __restrict__ vol, const double* __restrict__ X, const T* __restrict__ k, int64_t kstride,
                 const T* __restrict__ Tf, const int32_t* __restrict__ pos, T* __restrict__ ebuf, T* __restrict__ W) {
    constexpr int NV = D + 1;
    const int nq = min(HT_SC, S - s0);
    for (int e = blockIdx.x * HT_NT + threadIdx.x; e < E; e += gridDim.x * HT_NT) {
        int c[NV];
#pragma unroll
        for (int a = 0; a < NV; ++a) c[a] = __ldg(conn + (int64_t)e * NV + a);
        T g[D][D];
        T Ve;
        if constexpr (OTF) {
            geometry_of<D, T>(X, c, g, Ve);
        } else {
#pragma unroll
            for (int b = 0; b < D; ++b)
#pragma unroll
                for (int j = 0; j < D; ++j) g[b][j] = __ldg(grad + (int64_t)(b * D + j) * E + e);
            Ve = __ldg(vol + e);
        }
        const T kv = __ldg(k + (int64_t)e * kstride) * Ve;
        T fl[NV][HT_SC];
#pragma unroll
        for (int sq = 0; sq < HT_SC; ++sq) {
            T gT[D];
            if (sq < nq) {
                const T* Ts = Tf + (int64_t)(s0 + sq) * sstride;
                const T t0 = __ldg(Ts + c[0]);
                T dt[D];
#pragma unroll
                for (int b = 0; b < D; ++b) dt[b] = __ldg(Ts + c[b + 1]) - t0;
                T gg = T(0);
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    T v = dt[0] * g[0][j];
#pragma unroll
                    for (int b = 1; b < D; ++b) v = fma(dt[b], g[b][j], v);
                    gg = j == 0 ? v * v : fma(v, v, gg);
                    gT[j] = v * kv;
                }
                if (W) W[(int64_t)(s0 + sq) * E + e] = (T(0.5) * kv) * gg;   // the same W_e as k_heat_elem
            } else {
#pragma unroll
                for (int j = 0; j < D; ++j) gT[j] = T(0);
            }
            // vertex a >= 1: kV grad T . grad N_a; vertex 0: minus their sum
            T f0 = T(0);
#pragma unroll
            for (int b = 0; b < D; ++b) {
                T v = gT[0] * g[b][0];
#pragma unroll
                for (int j = 1; j < D; ++j) v = fma(gT[j], g[b][j], v);
                fl[b + 1][sq] = v;
                f0 -= v;
            }
            fl[0][sq] = f0;
        }
#pragma unroll
        for (int a = 0; a < NV; ++a) {
            T* dst = ebuf + (int64_t)__ldg(pos + (int64_t)e * NV + a) * HT_SC;
            if constexpr (sizeof(T) == 4 && HT_SC == 4) {
                *reinterpret_cast<float4*>(dst) = make_float4(fl[a][0], fl[a][1], fl[a][2], fl[a][3]);
            } else {
#pragma unroll
                for (int sq = 0; sq < HT_SC; ++sq) dst[sq] = fl[a][sq];
            }
        }
    }
}

template <class T>
__global__ void __launch_bounds__(HT_NT)
k_heat_node_sum(int N, int S, int s0, int64_t sstride, const int32_t* __restrict__ csr_ptr, const T* __restrict__ ebuf,
                T* __restrict__ r, unsigned long long* __restrict__ stamp, unsigned long long key) {
    const int nq = min(HT_SC, S - s0);
    if (blockIdx.x == 0 && threadIdx.x == 0) *stamp = key;   // positions complete (previous kernel)
    for (int n = blockIdx.x * HT_NT + threadIdx.x; n < N; n += gridDim.x * HT_NT) {
        T acc[HT_SC];
#pragma unroll
        for (int sq = 0; sq < HT_SC; ++sq) acc[sq] = T(0);
        for (int q = __ldg(csr_ptr + n); q < __ldg(csr_ptr + n + 1); ++q) {
            if constexpr (sizeof(T) == 4 && HT_SC == 4) {
                const float4 v = __ldcs(reinterpret_cast<const float4*>(ebuf + (int64_t)q * HT_SC));
                acc[0] += v.x; acc[1] += v.y; acc[2] += v.z; acc[3] += v.w;
            } else {
#pragma unroll
                for (int sq = 0; sq < HT_SC; ++sq) acc[sq] += ebuf[(int64_t)q * HT_SC + sq];
            }
        }
#pragma unroll
        for (int sq = 0; sq < HT_SC; ++sq)
            if (sq < nq) r[(int64_t)(s0 + sq) * sstride + n] = acc[sq];
    }
}

size_t heat_ec_bytes(const pfem_mesh* m) {
    const size_t nnz = (size_t)m->n_elems * (m->dim + 1);
    const size_t ts = m->dtype == PFEM_F64 ? 8 : 4;
    return 256 + ((sizeof(int32_t) * nnz + 255) / 256 * 256) + ts * nnz * HT_SC;   // stamp | pos | entries
}

template <int D, class T>
pfem_status heat_impl(const pfem_mesh* m, const void* k, int64_t kstride, int S, const void* Tf, int64_t sstride,
                      const void* f, void* W, void* totals, void* r, void* ws, int otf, cudaStream_t s) {
    double* partial = ws ? (double*)((char*)ws + heat_ec_bytes(m)) : nullptr;
    const int E = m->n_elems, N = m->n_nodes;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const bool ec = r && ws;   // element-centric fluxes through a CSR-ordered entry buffer (W_e formed in the same pass)
    if (W && !ec) {
        const int g = std::max(1, std::min(8 * nsm, (E + HT_NT - 1) / HT_NT));
        k_heat_elem<D, T><<<g, HT_NT, 0, s>>>(E, N, S, sstride, m->conn, (const T*)m->grad, (const T*)m->vol,
                                              (const T*)k, kstride, (const T*)Tf, (T*)W);
        PFEM_LAUNCH_CHECK("k_heat_elem");
        count_launch();
    }
    if (ec) {
        // element-centric: per-element vertex fluxes at their CSR entries, node sums in CSR order
        char* w = (char*)ws;   // fixed offset 0, independent of S
        // the CSR entry positions depend only on the mesh: computed once per (workspace, plan)
        unsigned long long* stamp = (unsigned long long*)w;
        // (never 0, so a zero-filled workspace always computes them; splitmix64 of the serial)
        unsigned long long key = reinterpret_cast<const Plan*>(m->plan)->serial + 0x9E3779B97F4A7C15ull;
        key = (key ^ (key >> 30)) * 0xBF58476D1CE4E5B9ull;
        key = (key ^ (key >> 27)) * 0x94D049BB133111EBull;
        key = (key ^ (key >> 31)) | 1ull;
        w += 256;
        int32_t* pos = (int32_t*)w;
        const int64_t nnz = (int64_t)E * (D + 1);
        T* ebuf = (T*)(w + ((sizeof(int32_t) * (size_t)nnz + 255) / 256 * 256));
        const int gp = (int)std::max<int64_t>(1, std::min<int64_t>(8 * nsm, (nnz + HT_NT - 1) / HT_NT));
        k_heat_entry_pos<<<gp, HT_NT, 0, s>>>(nnz, m->csr_ent, pos, stamp, key);
        PFEM_LAUNCH_CHECK("k_heat_entry_pos");
        count_launch();
        const int ge = std::max(1, std::min(16 * nsm, (E + HT_NT - 1) / HT_NT));
        const int gn = std::max(1, std::min(16 * nsm, (N + HT_NT - 1) / HT_NT));
        for (int s0 = 0; s0 < S; s0 += HT_SC) {
            if (otf)
                k_heat_elem_flux<D, T, true><<<ge, HT_NT, 0, s>>>(E, S, s0, sstride, m->conn, (const T*)m->grad,
                                                                  (const T*)m->vol, m->coords, (const T*)k, kstride,
                                                                  (const T*)Tf, pos, ebuf, (T*)W);
            else
                k_heat_elem_flux<D, T, false><<<ge, HT_NT, 0, s>>>(E, S, s0, sstride, m->conn, (const T*)m->grad,
                                                                   (const T*)m->vol, m->coords, (const T*)k, kstride,
                                                                   (const T*)Tf, pos, ebuf, (T*)W);
            PFEM_LAUNCH_CHECK("k_heat_elem_flux");
            k_heat_node_sum<T><<<gn, HT_NT, 0, s>>>(N, S, s0, sstride, m->csr_ptr, ebuf, (T*)r, stamp, key);
            PFEM_LAUNCH_CHECK("k_heat_node_sum");
            count_launch(2);
        }
    }
    if (totals) {
        const int K = m->n_parts;
        k_heat_partials<T><<<dim3(HT_SLICES, K, S), HT_NT, 0, s>>>(E, N, K, sstride, m->part_elem, m->part_node,
                                                                    (const T*)W, (const T*)f, (const T*)Tf, partial);
        PFEM_LAUNCH_CHECK("k_heat_partials");
        k_heat_totals<T><<<(S * K + HT_NT - 1) / HT_NT, HT_NT, 0, s>>>(S * K, partial, (T*)totals);
        PFEM_LAUNCH_CHECK("k_heat_totals");
        count_launch(2);
    }
    if (r && !ec) {
        const int g = std::max(1, std::min(8 * nsm, (N + HT_NT - 1) / HT_NT));
        k_heat_flux<D, T><<<g, HT_NT, 0, s>>>(N, E, S, sstride, m->csr_ptr, m->csr_ent, m->conn, (const T*)m->grad,
                                              (const T*)m->vol, (const T*)k, kstride, (const T*)Tf, (T*)r);
        PFEM_LAUNCH_CHECK("k_heat_flux");
        count_launch();
    }
    return PFEM_OK;
}

pfem_status run_heat(const pfem_mesh* m, const void* k, int64_t kstride, int S, const void* Tf, int64_t sstride,
                     const void* f, void* W, void* totals, void* r, void* ws, int otf, cudaStream_t s) {
    if (m->dim == 2)
        return m->dtype == PFEM_F32 ? heat_impl<2, float>(m, k, kstride, S, Tf, sstride, f, W, totals, r, ws, otf, s)
                                    : heat_impl<2, double>(m, k, kstride, S, Tf, sstride, f, W, totals, r, ws, otf, s);
    return m->dtype == PFEM_F32 ? heat_impl<3, float>(m, k, kstride, S, Tf, sstride, f, W, totals, r, ws, otf, s)
                                : heat_impl<3, double>(m, k, kstride, S, Tf, sstride, f, W, totals, r, ws, otf, s);
}

}  // namespace pfem

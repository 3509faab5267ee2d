// assemble.cuh — the fused element kernel of the hot path (§8 rows a2-a6), CSR mode.
//
// One CTA per element block (contiguous element range of <= eb_max elements, taken in
// ticket order).  For each chunk of ST samples:
//   phase 1 (thread per element): gather u (or v), H, P / dP, psi, element forces
//           -> shared memory fbuf[ST][d][d+1][eb_max]; W_e; per-sample energy sums
//   phase 2 (thread per (occurrence, sample)): every node touched by the block sums its
//           block-local CSR entries (ascending element, slot) from fbuf.
//           owner nodes write the output; nodes owned by a later block write a partial.
// Then the block publishes its partials (flag = epoch+1), waits for the earlier blocks
// holding partials of nodes it owns, and adds them (ascending block order) to its own
// segment.  Every sum has a fixed order: no float atomics anywhere (north star).
// Per-block energy / f.u / dot sums are reduced hierarchically: the last block of each
// chunk of CHUNK blocks reduces the chunk, the last block overall reduces the chunks per
// part and writes the totals (and, for CG, alpha = rho / p.q).
#pragma once

#include "common.cuh"
#include "element.cuh"

namespace pfem {

enum { OP_ENERGY = 0, OP_ENERGY_RESIDUAL = 1, OP_RESIDUAL = 2, OP_TANGENT = 3 };
constexpr int ASM_NT = 256;
constexpr int CHUNK = 32;     // blocks per reduction chunk

struct CgState {
    double rho, rho_new, alpha, beta, bnorm2, tol2, pq, pad0;
    int32_t k, max_iter, done, status;   // status: 0 running, 1 converged, 2 breakdown, 3 max_iter
    int32_t pad[4];
};

template <class T>
struct AsmParams {
    int E, N, S, K;
    int64_t sstride;
    const int32_t* conn;
    const T* grad;
    const T* vol;
    MatArgs<T> mat;
    const T* u;            // field (energy / residual) or NH state (tangent)
    const T* v;            // tangent direction
    const uint8_t* mask;   // tangent Dirichlet mask (nullable)
    const T* f_ext;        // nullable
    T* W_e;                // nullable [S][E]
    T* totals;             // nullable [S][K]
    T* out;                // residual / Kv (nullable for OP_ENERGY)
    pfem_flags* uflags;    // nullable
    // plan
    int n_blocks, n_occ, eb_max, n_chunks;
    const int32_t* blk_elem;
    const int32_t* blk_chunk;
    const int32_t* chunk_blk;
    const int32_t* part_chunk;
    const int32_t* blk_occ;
    const int32_t* blk_min_dep;
    const int32_t* part_blk;
    const int32_t* occ_node;
    const int32_t* occ_ent_ptr;
    const uint16_t* loc_ent;
    const int32_t* node_occ_ptr;
    const int32_t* node_occ;
    // workspace
    Counters* ctr;
    int32_t* flag;         // [n_blocks]
    double* blk_sum;       // [R][n_blocks], R = 2S (+1 for the CG dot)
    int32_t* chunk_done;   // [n_chunks]
    double* chunk_sum;     // [R][n_chunks]
    T* partial;            // [S][n_occ][D]
    CgState* cg;           // non-null: fused p.q and alpha epilogue (S == 1)
};

// deterministic CTA reduction of one double per thread (fixed shuffle tree + fixed order)
template <int NT>
__device__ __forceinline__ double cta_sum(double v, double* sred) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sred[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < NT / 32; ++i) r += sred[i];
    return r;   // valid in thread 0
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int D, int MODEL, class T, int OP, int ST, bool MASKED>
__global__ void __launch_bounds__(ASM_NT)
k_assemble(const AsmParams<T> p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* fbuf = reinterpret_cast<T*>(smem_raw);
    __shared__ int s_b, s_epoch, s_last, s_chunk_last;
    __shared__ double s_red[ASM_NT / 32];
    constexpr bool HAS_FORCE = OP != OP_ENERGY;
    constexpr bool HAS_PSI = OP == OP_ENERGY || OP == OP_ENERGY_RESIDUAL;
    constexpr int NV = D + 1;
    const int tid = threadIdx.x;
    if (p.cg && ld_relaxed_i(&p.cg->done)) return;     // converged CG: whole grid exits

    if (tid == 0) {
        s_b = atomicAdd(&p.ctr->ticket, 1);
        s_epoch = ld_relaxed_i(&p.ctr->epoch);
    }
    __syncthreads();
    const int b = s_b, epoch = s_epoch;
    const int e0 = p.blk_elem[b], e1 = p.blk_elem[b + 1], ne = e1 - e0;
    const int o0 = p.blk_occ[b], no = p.blk_occ[b + 1] - o0;
    const int EBM = p.eb_max;
    const int S = p.S;
    int n_inv = 0, first_inv = INT32_MAX, n_nonfin = 0;
    double dot_acc = 0.0;

    for (int s0 = 0; s0 < S; s0 += ST) {
        // ---------------- phase 1: elements
        T wacc[ST];
#pragma unroll
        for (int q = 0; q < ST; ++q) wacc[q] = T(0);
        for (int el = tid; el < ne; el += ASM_NT) {
            const int e = e0 + el;
            Geo<D, T> G;
            load_geo<D, T>(e, p.E, p.conn, p.grad, p.vol, p.mat, G);
#pragma unroll
            for (int q = 0; q < ST; ++q) {
                const int s = s0 + q;
                if (ST > 1 && s >= S) break;
                T x[NV][D], H[D][D], P[D][D], psi = T(0);
                bool bad = false;
                if (OP == OP_TANGENT) {
                    NhState<D, T> NS;
                    if (MODEL == MODEL_NH) {
                        T Hu[D][D], H2[D][D];
                        gather<D, T, false>(p.u + (int64_t)s * p.sstride, nullptr, G, x);
                        grad_of<D, T>(G, x, Hu);
                        nh_state<D, T>(Hu, NS, H2);
                        bad = !(NS.x > T(-1));
                    }
                    gather<D, T, MASKED>(p.v + (int64_t)s * p.sstride, p.mask, G, x);
                    grad_of<D, T>(G, x, H);
                    dstress<D, MODEL, T>(G, NS, H, P);
                } else {
                    gather<D, T, false>(p.u + (int64_t)s * p.sstride, nullptr, G, x);
                    grad_of<D, T>(G, x, H);
                    if (HAS_FORCE)
                        stress<D, MODEL, T, HAS_PSI>(G, H, P, psi, bad);
                    else {
                        T Pd[D][D];
                        stress<D, MODEL, T, true>(G, H, Pd, psi, bad);
                    }
                }
                if (MODEL == MODEL_NH && bad) {
                    ++n_inv;
                    first_inv = min(first_inv, e);
                }
                if (HAS_PSI) {
                    const T W = G.V * psi;
                    if (!isfinite(W)) ++n_nonfin;
                    wacc[q] += W;
                    if (p.W_e) p.W_e[(int64_t)s * p.E + e] = W;
                }
                if (HAS_FORCE) {
                    T f[NV][D];
                    forces<D, T>(G, P, f);
#pragma unroll
                    for (int i = 0; i < D; ++i)
#pragma unroll
                        for (int a = 0; a < NV; ++a) fbuf[((q * D + i) * NV + a) * EBM + el] = f[a][i];
                    if (!HAS_PSI && !isfinite(f[0][0] + f[1][0])) ++n_nonfin;
                }
            }
        }
        if (HAS_PSI) {
#pragma unroll
            for (int q = 0; q < ST; ++q) {
                if (ST > 1 && s0 + q >= S) break;
                double t = cta_sum<ASM_NT>((double)wacc[q], s_red);
                if (tid == 0) p.blk_sum[(int64_t)(s0 + q) * p.n_blocks + b] = t;
            }
        }
        __syncthreads();
        // ---------------- phase 2: block-local CSR gather
        double fu[ST];
#pragma unroll
        for (int q = 0; q < ST; ++q) fu[q] = 0.0;
        const int nq = min(ST, S - s0);
        if (HAS_FORCE || p.f_ext) {
            for (int idx = tid; idx < no * nq; idx += ASM_NT) {
                const int q = idx / no;
                const int o = o0 + (idx - q * no);
                const int s = s0 + q;
                const int word = __ldg(p.occ_node + o);
                const int node = word & OCC_NODE_MASK;
                const int64_t nb = (int64_t)s * p.sstride + (int64_t)node * D;
                if (HAS_FORCE) {
                    T acc[D];
#pragma unroll
                    for (int i = 0; i < D; ++i) acc[i] = T(0);
                    const int k1 = __ldg(p.occ_ent_ptr + o + 1);
                    for (int k = __ldg(p.occ_ent_ptr + o); k < k1; ++k) {
                        const int j = __ldg(p.loc_ent + k);
                        const int el = j / NV, a = j - el * NV;
#pragma unroll
                        for (int i = 0; i < D; ++i) acc[i] += fbuf[((q * D + i) * NV + a) * EBM + el];
                    }
                    if (word & OCC_NONOWNER) {
                        T* dst = p.partial + ((int64_t)s * p.n_occ + o) * D;
#pragma unroll
                        for (int i = 0; i < D; ++i) dst[i] = acc[i];
                    } else {
                        const bool final_now = !(word & OCC_EARLIER);
#pragma unroll
                        for (int i = 0; i < D; ++i) {
                            T val = acc[i];
                            if (OP == OP_TANGENT && MASKED && final_now && __ldg(p.mask + (int64_t)node * D + i))
                                val = __ldg(p.v + nb + i);
                            p.out[nb + i] = val;
                            if (OP == OP_TANGENT && p.cg && final_now) dot_acc += (double)__ldg(p.v + nb + i) * (double)val;
                        }
                    }
                }
                if (HAS_PSI && p.f_ext && !(word & OCC_NONOWNER)) {
                    double w = 0.0;
#pragma unroll
                    for (int i = 0; i < D; ++i)
                        w += (double)__ldg(p.f_ext + (int64_t)node * D + i) * (double)__ldg(p.u + nb + i);
#pragma unroll
                    for (int qq = 0; qq < ST; ++qq)
                        if (qq == q) fu[qq] += w;
                }
            }
        }
        if (HAS_PSI) {
#pragma unroll
            for (int q = 0; q < ST; ++q) {
                if (ST > 1 && s0 + q >= S) break;
                double t = p.f_ext ? cta_sum<ASM_NT>(fu[q], s_red) : 0.0;
                if (tid == 0) p.blk_sum[(int64_t)(S + s0 + q) * p.n_blocks + b] = t;
            }
        }
        __syncthreads();
    }

    if (HAS_FORCE) {
        // ---------------- publish partials, wait for earlier blocks, fix up owned nodes
        __threadfence();
        __syncthreads();
        if (tid == 0) st_release_gpu(p.flag + b, epoch + 1);
        const int md = __ldg(p.blk_min_dep + b);
        if (md < b) {
            if (tid < 32) {
                for (int q = md + tid; q < b; q += 32) {
                    while (ld_acquire_gpu(p.flag + q) != epoch + 1) __nanosleep(32);
                }
                __syncwarp();
            }
            __syncthreads();
            for (int idx = tid; idx < no * S; idx += ASM_NT) {
                const int s = idx / no;
                const int o = o0 + (idx - s * no);
                const int word = __ldg(p.occ_node + o);
                if (!(word & OCC_EARLIER)) continue;
                const int node = word & OCC_NODE_MASK;
                const int64_t nb = (int64_t)s * p.sstride + (int64_t)node * D;
                T acc[D];
                const int k0 = __ldg(p.node_occ_ptr + node), k1 = __ldg(p.node_occ_ptr + node + 1) - 1;
                {
                    const T* src = p.partial + ((int64_t)s * p.n_occ + __ldg(p.node_occ + k0)) * D;
#pragma unroll
                    for (int i = 0; i < D; ++i) acc[i] = ld_relaxed(src + i);
                }
                for (int k = k0 + 1; k < k1; ++k) {
                    const T* src = p.partial + ((int64_t)s * p.n_occ + __ldg(p.node_occ + k)) * D;
#pragma unroll
                    for (int i = 0; i < D; ++i) acc[i] += ld_relaxed(src + i);
                }
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    T val = acc[i] + p.out[nb + i];
                    if (OP == OP_TANGENT && MASKED && __ldg(p.mask + (int64_t)node * D + i)) val = __ldg(p.v + nb + i);
                    p.out[nb + i] = val;
                    if (OP == OP_TANGENT && p.cg) dot_acc += (double)__ldg(p.v + nb + i) * (double)val;
                }
            }
        }
        if (OP == OP_TANGENT && p.cg) {
            double t = cta_sum<ASM_NT>(dot_acc, s_red);
            if (tid == 0) p.blk_sum[(int64_t)(2 * S) * p.n_blocks + b] = t;
        }
    }

    // ---------------- flags
    {
        // reduce the per-thread inversion counters through shared atomics (integers)
        __shared__ int s_ninv, s_first, s_nf;
        if (tid == 0) { s_ninv = 0; s_first = INT32_MAX; s_nf = 0; }
        __syncthreads();
        if (n_inv) { atomicAdd(&s_ninv, n_inv); atomicMin(&s_first, first_inv); }
        if (n_nonfin) atomicAdd(&s_nf, n_nonfin);
        __syncthreads();
        if (tid == 0) {
            if (s_ninv) { atomicAdd(&p.ctr->n_inv, s_ninv); atomicMax(&p.ctr->first_inv, INT32_MAX - s_first); }
            if (s_nf) atomicAdd(&p.ctr->n_nonfinite, s_nf);
        }
    }

    // ---------------- hierarchical reduction of the per-block sums
    // channels: [0, 2S) energy / f.u per sample (HAS_PSI), 2S: CG p.q (tangent + cg)
    const int rb = HAS_PSI ? 0 : 2 * S;
    const int re = (OP == OP_TANGENT && p.cg) ? 2 * S + 1 : (HAS_PSI ? 2 * S : 2 * S);
    __threadfence();
    __syncthreads();
    const int chunk = __ldg(p.blk_chunk + b);
    const int c0 = __ldg(p.chunk_blk + chunk), c1 = __ldg(p.chunk_blk + chunk + 1);
    if (tid == 0) s_chunk_last = (atomicAdd(p.chunk_done + chunk, 1) == (c1 - c0) - 1);
    __syncthreads();
    if (!s_chunk_last) return;
    __threadfence();
    {
        const int w = tid >> 5, l = tid & 31;
        for (int r = rb + w; r < re; r += ASM_NT / 32) {
            double v = (c0 + l < c1) ? ld_relaxed(p.blk_sum + (int64_t)r * p.n_blocks + c0 + l) : 0.0;
            v = warp_sum(v);
            if (l == 0) p.chunk_sum[(int64_t)r * p.n_chunks + chunk] = v;
        }
        if (tid == 0) p.chunk_done[chunk] = 0;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&p.ctr->done, 1) == p.n_chunks - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // ---------------- final: totals per (sample, part); CG alpha
    {
        const int w = tid >> 5, l = tid & 31;
        if (HAS_PSI && p.totals) {
            for (int pair = w; pair < S * p.K; pair += ASM_NT / 32) {
                const int s = pair / p.K, k = pair - s * p.K;
                const int cb = __ldg(p.part_chunk + k), ce = __ldg(p.part_chunk + k + 1);
                double wv = 0.0, fv = 0.0;
                for (int c = cb + l; c < ce; c += 32) {
                    wv += ld_relaxed(p.chunk_sum + (int64_t)s * p.n_chunks + c);
                    fv += ld_relaxed(p.chunk_sum + (int64_t)(S + s) * p.n_chunks + c);
                }
                wv = warp_sum(wv);
                fv = warp_sum(fv);
                if (l == 0) p.totals[(int64_t)s * p.K + k] = (T)(wv - fv);
            }
        }
        if (OP == OP_TANGENT && p.cg && w == 0) {
            double pq = 0.0;
            for (int c = l; c < p.n_chunks; c += 32) pq += ld_relaxed(p.chunk_sum + (int64_t)(2 * S) * p.n_chunks + c);
            pq = warp_sum(pq);
            if (l == 0) {
                CgState* cg = p.cg;
                cg->pq = pq;
                if (!(pq > 0.0)) {
                    cg->status = 2;
                    cg->done = 1;
                    cg->alpha = 0.0;
                } else {
                    cg->alpha = cg->rho / pq;
                }
            }
        }
        if (tid == 0) {
            const int ni = ld_relaxed_i(&p.ctr->n_inv);
            const int fi = ld_relaxed_i(&p.ctr->first_inv);
            if (p.uflags) {
                p.uflags->n_inverted = ni;
                p.uflags->first_inverted = fi == 0 ? -1 : (INT32_MAX - fi);
                p.uflags->n_nonfinite = ld_relaxed_i(&p.ctr->n_nonfinite);
                p.uflags->reserved = 0;
            }
            p.ctr->n_inv = 0;
            p.ctr->first_inv = 0;
            p.ctr->n_nonfinite = 0;
            p.ctr->done = 0;
            p.ctr->ticket = 0;
            __threadfence();
            p.ctr->epoch = epoch + 1;
        }
    }
}


// ====================================================================================
// COLOUR mode: colour-ordered scatter.  One launch per colour of the greedy colouring;
// no two elements of a colour share a node, so each (element, slot) does one plain
// read-modify-write of the output.  Summation order at a node: ascending colour.
// ====================================================================================
template <int D, int MODEL, class T, int OP, bool MASKED>
__global__ void __launch_bounds__(ASM_NT)
k_colour_pass(const AsmParams<T> p, const int32_t* __restrict__ colour_elems, int i0, int i1,
              T* __restrict__ wtmp) {
    constexpr bool HAS_FORCE = OP != OP_ENERGY;
    constexpr bool HAS_PSI = OP == OP_ENERGY || OP == OP_ENERGY_RESIDUAL;
    constexpr int NV = D + 1;
    const int i = i0 + blockIdx.x * ASM_NT + threadIdx.x;
    if (i >= i1) return;
    const int e = __ldg(colour_elems + i);
    Geo<D, T> G;
    load_geo<D, T>(e, p.E, p.conn, p.grad, p.vol, p.mat, G);
    int n_inv = 0, n_nonfin = 0;
    for (int s = 0; s < p.S; ++s) {
        T x[NV][D], H[D][D], P[D][D], psi = T(0);
        bool bad = false;
        if (OP == OP_TANGENT) {
            NhState<D, T> NS;
            if (MODEL == MODEL_NH) {
                T Hu[D][D], H2[D][D];
                gather<D, T, false>(p.u + (int64_t)s * p.sstride, nullptr, G, x);
                grad_of<D, T>(G, x, Hu);
                nh_state<D, T>(Hu, NS, H2);
                bad = !(NS.x > T(-1));
            }
            gather<D, T, MASKED>(p.v + (int64_t)s * p.sstride, p.mask, G, x);
            grad_of<D, T>(G, x, H);
            dstress<D, MODEL, T>(G, NS, H, P);
        } else {
            gather<D, T, false>(p.u + (int64_t)s * p.sstride, nullptr, G, x);
            grad_of<D, T>(G, x, H);
            stress<D, MODEL, T, true>(G, H, P, psi, bad);
        }
        if (MODEL == MODEL_NH && bad) ++n_inv;
        if (HAS_PSI) {
            const T W = G.V * psi;
            if (!isfinite(W)) ++n_nonfin;
            wtmp[(int64_t)s * p.E + e] = W;
        }
        if (HAS_FORCE) {
            T f[NV][D];
            forces<D, T>(G, P, f);
#pragma unroll
            for (int a = 0; a < NV; ++a)
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    T* dst = p.out + (int64_t)s * p.sstride + (int64_t)G.v[a] * D + k;
                    *dst = *dst + f[a][k];
                }
        }
    }
    if (n_inv) {
        atomicAdd(&p.ctr->n_inv, n_inv);
        atomicMax(&p.ctr->first_inv, INT32_MAX - e);
    }
    if (n_nonfin) atomicAdd(&p.ctr->n_nonfinite, n_nonfin);
}

// masked rows of the tangent output: (I-M) K (I-M) v + M v
template <int D, class T>
__global__ void k_mask_rows(int S, int N, int64_t sstride, const uint8_t* __restrict__ mask,
                            const T* __restrict__ v, T* __restrict__ out) {
    const int64_t n = (int64_t)N * D;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (!__ldg(mask + i)) return;
    for (int s = 0; s < S; ++s) out[(int64_t)s * sstride + i] = __ldg(v + (int64_t)s * sstride + i);
}

// per (sample, part) totals for the colour mode: fixed-order CTA reduction over the
// part's elements (W) and nodes (f.u); CTA 0 also reports and resets the flags.
template <int D, class T>
__global__ void __launch_bounds__(ASM_NT)
k_colour_totals(const AsmParams<T> p, const int32_t* __restrict__ part_elem,
                const int32_t* __restrict__ part_node, const T* __restrict__ wtmp, int want_totals) {
    __shared__ double s_red[ASM_NT / 32];
    const int pair = blockIdx.x;
    if (want_totals) {
        const int s = pair / p.K, k = pair - s * p.K;
        double w = 0.0;
        for (int e = part_elem[k] + threadIdx.x; e < part_elem[k + 1]; e += ASM_NT) w += (double)wtmp[(int64_t)s * p.E + e];
        if (p.f_ext)
            for (int64_t j = (int64_t)part_node[k] * D + threadIdx.x; j < (int64_t)part_node[k + 1] * D; j += ASM_NT)
                w -= (double)__ldg(p.f_ext + j) * (double)__ldg(p.u + (int64_t)s * p.sstride + j);
        const double t = cta_sum<ASM_NT>(w, s_red);
        if (threadIdx.x == 0) {
            p.totals[(int64_t)s * p.K + k] = (T)t;
            if (p.W_e) { /* elem energies were written to W_e directly (wtmp == W_e) */ }
        }
    }
    if (pair == 0 && threadIdx.x == 0) {
        const int ni = p.ctr->n_inv, fi = p.ctr->first_inv;
        if (p.uflags) {
            p.uflags->n_inverted = ni;
            p.uflags->first_inverted = fi == 0 ? -1 : (INT32_MAX - fi);
            p.uflags->n_nonfinite = p.ctr->n_nonfinite;
            p.uflags->reserved = 0;
        }
        p.ctr->n_inv = 0;
        p.ctr->first_inv = 0;
        p.ctr->n_nonfinite = 0;
    }
}

}  // namespace pfem

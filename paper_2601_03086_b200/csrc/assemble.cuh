// assemble.cuh — the fused element kernels of the hot path (§8 rows a2-a6).
//
// CSR mode (the reported path).  The plan (prep.cu) cuts the elements into blocks of at
// most EB consecutive elements.  A persistent grid (resident CTAs) loops over tickets
// (atomic counter, so every awaited block is held by a running CTA); the ticket after next
// is requested and the next block's element arrays (conn, grad N, V, material) are
// prefetched into shared memory with cp.async while the current block computes.
// Ticket t:
//   main (t < n_blocks), block b = t:
//     phase 1, thread per element: gather u (or v), H, P / dP, psi; the d+1 nodal force
//       vectors of all ST samples -> shared fbuf[slot][element][dim][sample] (fp32 samples
//       are processed in FFMA2 pairs and stored as float2); W_e; per-sample energy sums
//     phase 2, thread per node occurrence of the block: sum the block-local CSR entries
//       (ascending element, slot) with vector loads of all ST samples at once.
//       owner nodes without earlier partials: final value; owners with earlier partials:
//       own segment (fixed up later); nodes owned by a later block: partial.
//     publish: flag[b] = epoch + 1.
//   lagged fix-up (t >= L), block c = t - L: for every owned node of c that has partials
//     in earlier blocks: out = ((p_1 + p_2) + ...) + own, ascending block order.  The lag L
//     (= resident CTAs) makes the awaited flags (blocks [min_dep(c), c]) almost always
//     already set, so CTAs do not idle on dependencies.
// Every sum has a fixed order: no floating-point atomics anywhere (north star); the
// result is independent of scheduling and bitwise reproducible.
// Reductions (energies, f.u, CG p.q): per block -> per chunk (<= 32 blocks of one part,
// reduced by the CTA completing the chunk's 2 arrivals per block) -> per part (the CTA
// completing the last chunk; it also writes CG alpha and resets the workspace counters).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "element.cuh"

namespace pfem {

enum { OP_ENERGY = 0, OP_ENERGY_RESIDUAL = 1, OP_RESIDUAL = 2, OP_TANGENT = 3 };
constexpr int ASM_NT = 256;   // main (element / occurrence) threads per CTA
constexpr int FIX_WARPS = 2;  // fix-up warps per CTA
constexpr int CHUNK = 32;     // blocks per reduction chunk (== CHUNK_BLOCKS of prep.cu)

template <int D>
struct EbOf {
    static constexpr int value = D == 3 ? 256 : 512;   // compile-time block capacity
};

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
    int n_blocks, n_occ, eb_max, n_chunks, lag;
    int dbg;               // experiment switches (PFEM_DEBUG env): 1 no phase-1 math, 2 no phase 2, 4 no fix-up, 8 no sums, 16 no staging
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
    const int32_t* blk_fix;
    const int32_t* fix_occ;
    const int32_t* fix_node;
    const int32_t* fix_src_ptr;
    const int32_t* fix_src;
    RecLayout rec;
    const unsigned char* recs;
    // workspace
    Counters* ctr;
    int32_t* flag;         // [n_blocks]
    double* blk_sum;       // [2S+2][n_blocks]: W_s, f.u_s, dot(main), dot(fix-up)
    int32_t* chunk_done;   // [n_chunks]
    double* chunk_sum;     // [2S+1][n_chunks]
    T* partial;            // [n_occ][S][D]
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

__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

template <class T>
__device__ __forceinline__ T warp_sum_t(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// vector load / store of N contiguous T in shared memory (N*sizeof(T) in {4..48} bytes)
template <class T, int N>
__device__ __forceinline__ void sld(const T* p, T* v) {
    if constexpr (sizeof(T) * N % 16 == 0) {
#pragma unroll
        for (int k = 0; k < N * (int)sizeof(T) / 16; ++k) {
            float4 q = reinterpret_cast<const float4*>(p)[k];
            memcpy(reinterpret_cast<char*>(v) + 16 * k, &q, 16);
        }
    } else if constexpr (sizeof(T) * N % 8 == 0) {
#pragma unroll
        for (int k = 0; k < N * (int)sizeof(T) / 8; ++k) {
            float2 q = reinterpret_cast<const float2*>(p)[k];
            memcpy(reinterpret_cast<char*>(v) + 8 * k, &q, 8);
        }
    } else {
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = p[k];
    }
}

template <class T, int N>
__device__ __forceinline__ void sst(T* p, const T* v) {
    if constexpr (sizeof(T) * N % 16 == 0) {
#pragma unroll
        for (int k = 0; k < N * (int)sizeof(T) / 16; ++k) {
            float4 q;
            memcpy(&q, reinterpret_cast<const char*>(v) + 16 * k, 16);
            reinterpret_cast<float4*>(p)[k] = q;
        }
    } else if constexpr (sizeof(T) * N % 8 == 0) {
#pragma unroll
        for (int k = 0; k < N * (int)sizeof(T) / 8; ++k) {
            float2 q;
            memcpy(&q, reinterpret_cast<const char*>(v) + 8 * k, 8);
            reinterpret_cast<float2*>(p)[k] = q;
        }
    } else {
#pragma unroll
        for (int k = 0; k < N; ++k) p[k] = v[k];
    }
}

// one chunk arrival; returns true (in all threads) if this CTA completed the chunk and
// must reduce it
__device__ __forceinline__ bool chunk_arrive(int* chunk_done, int ch, int need, int* s_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        *s_flag = (atomicAdd(chunk_done + ch, 1) == need - 1);
    }
    __syncthreads();
    return *s_flag != 0;
}

// ------------------------------------------------------------------ TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LAB_WAIT;\n"
        "}\n" ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}

template <int N>
__device__ __forceinline__ void cpn(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_addr(dst)), "l"(src), "n"(N));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void bar_main(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }

template <class T, int N>
__device__ __forceinline__ void ld_relaxed_vec(const T* p, T* v) {
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = ld_relaxed(p + k);
}

// stage block b: one bulk copy of its packed record (thread 0) + per-element material
// (cp.async, only for element-wise parameters); every thread commits one cp.async group
template <int D, class T, int NT>
__device__ __forceinline__ void stage_block(unsigned char* st, T* mst, uint64_t* bar, const AsmParams<T>& p, int b) {
    if (threadIdx.x == 0) {
        fence_proxy_async();   // earlier generic reads of this buffer precede the async write
        mbar_expect_tx(bar, p.rec.bytes);
        tma_bulk_g2s(st, p.recs + (size_t)b * p.rec.bytes, p.rec.bytes, bar);
    }
    if (p.mat.s0 | p.mat.s1) {
        const int e0 = __ldg(p.blk_elem + b), ne = __ldg(p.blk_elem + b + 1) - e0;
        for (int el = threadIdx.x; el < ne; el += NT) {
            if (p.mat.s0) cpn<sizeof(T)>(mst + el, p.mat.p0 + (int64_t)(e0 + el) * p.mat.s0);
            if (p.mat.s1) cpn<sizeof(T)>(mst + p.rec.eb + el, p.mat.p1 + (int64_t)(e0 + el) * p.mat.s1);
        }
    }
    cp_commit();
}

// warp-group reduction of the chunk containing block `blk` once all its arrivals are in;
// the completing group also finalises (totals / CG alpha) after the last chunk
template <class T>
__device__ __forceinline__ void chunk_reduce(const AsmParams<T>& p, int ch, int rb, int re, int w, int nw, int lane,
                                             bool& last) {
    const int c0 = __ldg(p.chunk_blk + ch), c1 = __ldg(p.chunk_blk + ch + 1);
    const int S = p.S;
    for (int r = rb + w; r < re; r += nw) {
        double v = 0.0;
        if (c0 + lane < c1) {
            v = ld_relaxed(p.blk_sum + (int64_t)r * p.n_blocks + c0 + lane);
            if (r == 2 * S) v += ld_relaxed(p.blk_sum + (int64_t)(2 * S + 1) * p.n_blocks + c0 + lane);
        }
        v = warp_sum(v);
        if (lane == 0) p.chunk_sum[(int64_t)r * p.n_chunks + ch] = v;
    }
    last = false;
    (void)c1;
}

template <class T, bool HAS_PSI, bool TANGENT>
__device__ __forceinline__ void finalize(const AsmParams<T>& p, int w, int nw, int lane) {
    const int S = p.S;
    if (HAS_PSI && p.totals) {
        for (int pair = w; pair < S * p.K; pair += nw) {
            const int s = pair / p.K, k = pair - s * p.K;
            const int cb = __ldg(p.part_chunk + k), ce = __ldg(p.part_chunk + k + 1);
            double wv = 0.0, fv = 0.0;
            for (int cc = cb + lane; cc < ce; cc += 32) {
                wv += ld_relaxed(p.chunk_sum + (int64_t)s * p.n_chunks + cc);
                fv += ld_relaxed(p.chunk_sum + (int64_t)(S + s) * p.n_chunks + cc);
            }
            wv = warp_sum(wv);
            fv = warp_sum(fv);
            if (lane == 0) p.totals[(int64_t)s * p.K + k] = (T)(wv - fv);
        }
    }
    if (TANGENT && p.cg && w == 0) {
        double pq = 0.0;
        for (int cc = lane; cc < p.n_chunks; cc += 32) pq += ld_relaxed(p.chunk_sum + (int64_t)(2 * S) * p.n_chunks + cc);
        pq = warp_sum(pq);
        if (lane == 0) {
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
}

// Persistent, software-pipelined CSR-mode kernel.
//   main warps (NT threads): ticket stream over blocks.  Per block: the packed record is
//     staged by ONE TMA bulk copy (prefetched one block ahead, mbarrier completion) and the
//     ticket after next is requested; phase 1 -> fbuf -> phase 2 -> outputs / partials;
//     warp 0 then publishes the block (flag, release) and does the reductions while the
//     other warps start the next block.  Main warps never wait on other CTAs.
//   fix-up warps (NFW x 32 threads): an independent ticket stream over blocks c; wait
//     until the blocks holding c's segments have published, then write the final value of
//     every node c owns that has earlier segments (ascending block order).
template <int D, int MODEL, class T, int OP, int ST, bool MASKED, int EB, int NT, int NFW>
__global__ void __launch_bounds__(NT + 32 * NFW, 2)
k_assemble(const AsmParams<T> p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* stage_ptr[2] = {smem_raw, smem_raw + p.rec.bytes};
    T* mstage = reinterpret_cast<T*>(smem_raw + 2 * (size_t)p.rec.bytes);               // [2][2][EB]
    T* fbuf = mstage + 4 * EB;                                                           // [NV][EB][D][ST]
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ int s_tk[2], s_epoch;
    __shared__ double s_red[NT / 32][2 * ST + 1];
    constexpr bool HAS_FORCE = OP != OP_ENERGY;
    constexpr bool HAS_PSI = OP == OP_ENERGY || OP == OP_ENERGY_RESIDUAL;
    constexpr int NV = D + 1;
    constexpr int SD = ST * D;
    using V = std::conditional_t<(sizeof(T) == 4 && ST % 2 == 0), F2, T>;
    constexpr int L = VTraits<V>::L;
    using A2 = std::conditional_t<(sizeof(T) == 4 && SD % 2 == 0), F2, T>;     // phase-2 accumulator
    constexpr int LA = VTraits<A2>::L;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int S = p.S;
    const bool cgdot = OP == OP_TANGENT && p.cg != nullptr;
    const int arrivals = cgdot ? 2 : 1;   // main (+ fix-up for the CG dot)
    if (p.cg && ld_relaxed_i(&p.cg->done)) return;     // converged CG: the whole grid exits

    if (tid == 0) {
        s_epoch = ld_relaxed_i(&p.ctr->epoch);
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const int epoch = s_epoch;
    int n_inv = 0, first_inv = INT32_MAX, n_nonfin = 0;

    if (warp >= NT / 32) {
        // =================================================================  fix-up warps
        if (!HAS_FORCE || (p.dbg & 4)) goto done;
        while (true) {
            int c = 0;
            if (lane == 0) c = atomicAdd(&p.ctr->fix_ticket, 1);
            c = __shfl_sync(0xffffffffu, c, 0);
            if (c >= p.n_blocks) break;
            double dot_acc = 0.0;
            const int f0 = __ldg(p.blk_fix + c), nfix = __ldg(p.blk_fix + c + 1) - f0;
            if (nfix > 0) {
                const int md = __ldg(p.blk_min_dep + c);
                for (int q = md + lane; q <= c; q += 32) {
                    unsigned ns = 256;
                    while (ld_relaxed_i(p.flag + q) != epoch + 1) {
                        __nanosleep(ns);
                        ns = min(ns * 2, 4096u);
                    }
                }
                __syncwarp();
                for (int fi = lane; fi < nfix; fi += 32) {
                    const int f = f0 + fi;
                    const int node = __ldg(p.fix_node + f);
                    const int k0 = __ldg(p.fix_src_ptr + f), k1 = __ldg(p.fix_src_ptr + f + 1);
                    for (int s = 0; s < S; ++s) {
                        T acc[D];
                        ld_relaxed_vec<T, D>(p.partial + ((int64_t)__ldg(p.fix_src + k0) * S + s) * D, acc);
                        for (int k = k0 + 1; k < k1; ++k) {
                            T v[D];
                            ld_relaxed_vec<T, D>(p.partial + ((int64_t)__ldg(p.fix_src + k) * S + s) * D, v);
#pragma unroll
                            for (int i = 0; i < D; ++i) acc[i] += v[i];
                        }
                        const int64_t nb = (int64_t)s * p.sstride + (int64_t)node * D;
#pragma unroll
                        for (int i = 0; i < D; ++i) {
                            T val = acc[i];
                            if (OP == OP_TANGENT && MASKED && __ldg(p.mask + (int64_t)node * D + i)) val = __ldg(p.v + nb + i);
                            p.out[nb + i] = val;
                            if (cgdot) dot_acc += (double)__ldg(p.v + nb + i) * (double)val;
                        }
                    }
                }
            }
            if (cgdot) {
                dot_acc = warp_sum(dot_acc);
                int last = 0;
                const int ch = __ldg(p.blk_chunk + c);
                if (lane == 0) {
                    p.blk_sum[(int64_t)(2 * S + 1) * p.n_blocks + c] = dot_acc;
                    const int need = arrivals * (__ldg(p.chunk_blk + ch + 1) - __ldg(p.chunk_blk + ch));
                    last = atom_add_acq_rel(p.chunk_done + ch, 1) == need - 1;
                }
                last = __shfl_sync(0xffffffffu, last, 0);
                if (last) {
                    bool dummy;
                    chunk_reduce<T>(p, ch, 2 * S, 2 * S + 1, 0, 1, lane, dummy);
                    int fin = 0;
                    if (lane == 0) {
                        p.chunk_done[ch] = 0;
                        fin = atom_add_acq_rel(&p.ctr->done, 1) == p.n_chunks - 1;
                    }
                    fin = __shfl_sync(0xffffffffu, fin, 0);
                    if (fin) finalize<T, HAS_PSI, OP == OP_TANGENT>(p, 0, 1, lane);
                }
            }
        }
        goto done;
    }

    {
        // =================================================================  main warps
        if (tid == 0) {
            s_tk[0] = atomicAdd(&p.ctr->ticket, 1);
            s_tk[1] = atomicAdd(&p.ctr->ticket, 1);
        }
        bar_main(NT);
        int t = s_tk[0], t_next = s_tk[1];
        uint32_t parity[2] = {0u, 0u};
        if (t < p.n_blocks && !(p.dbg & 16)) stage_block<D, T, NT>(stage_ptr[0], mstage, &s_bar[0], p, t);
        else cp_commit();
        int it = 0;
        int req = 0;   // ticket requested by thread 0 this iteration (consumed after phase 2)
        while (t < p.n_blocks) {
            const int cur = it & 1;
            if (tid == 0) req = (t_next < p.n_blocks) ? atomicAdd(&p.ctr->ticket, 1) : p.n_blocks;
            if (t_next < p.n_blocks && !(p.dbg & 16))
                stage_block<D, T, NT>(stage_ptr[cur ^ 1], mstage + 2 * EB * (cur ^ 1), &s_bar[cur ^ 1], p, t_next);
            else
                cp_commit();
            const int b = t;
            const int e0 = __ldg(p.blk_elem + b), ne = __ldg(p.blk_elem + b + 1) - e0;
            const int o0 = __ldg(p.blk_occ + b), no = __ldg(p.blk_occ + b + 1) - o0;
            const unsigned char* sg = stage_ptr[cur];
            const int32_t* sconn = reinterpret_cast<const int32_t*>(sg + p.rec.conn);
            const T* sgrad = reinterpret_cast<const T*>(sg + p.rec.g);
            const T* svol = reinterpret_cast<const T*>(sg + p.rec.vol);
            const int32_t* socc = reinterpret_cast<const int32_t*>(sg + p.rec.occ_node);
            const uint16_t* soe = reinterpret_cast<const uint16_t*>(sg + p.rec.occ_ent);
            const uint16_t* sle = reinterpret_cast<const uint16_t*>(sg + p.rec.loc_ent);
            const T* smat = mstage + 2 * EB * cur;
            cp_wait<1>();                                   // this thread's material copies
            if (!(p.dbg & 16)) mbar_wait(&s_bar[cur], parity[cur]);   // the block record
            parity[cur] ^= 1u;
            double dot_acc = 0.0;
            double wsum[ST], fsum[ST];
#pragma unroll
            for (int q = 0; q < ST; ++q) wsum[q] = fsum[q] = 0.0;
            for (int s0 = 0; s0 < S; s0 += ST) {
                const int nq = min(ST, S - s0);
                // ---------------- phase 1: elements
                T wacc[ST];
#pragma unroll
                for (int q = 0; q < ST; ++q) wacc[q] = T(0);
                for (int el = tid; el < ne; el += NT) {
                    const int e = e0 + el;
                    Geo<D, T> G;
                    if constexpr (D == 3) {
                        const int4 cv = *reinterpret_cast<const int4*>(sconn + el * 4);
                        G.v[0] = cv.x; G.v[1] = cv.y; G.v[2] = cv.z; G.v[3] = cv.w;
                    } else {
#pragma unroll
                        for (int a = 0; a <= D; ++a) G.v[a] = sconn[el * NV + a];
                    }
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int j = 0; j < D; ++j) G.g[a][j] = sgrad[(a * D + j) * EB + el];
                    G.V = svol[el];
                    {
                        const T m0 = p.mat.s0 ? smat[el] : __ldg(p.mat.p0);
                        const T m1 = p.mat.s1 ? smat[EB + el] : __ldg(p.mat.p1);
                        lame_of<T>(p.mat.kind, m0, m1, G.mu, G.lam);
                        G.mu *= G.V;
                        G.lam *= G.V;
                    }
#pragma unroll
                    for (int qq = 0; qq < ST; qq += L) {
                        if (qq >= nq || (p.dbg & 1)) break;
                        const int s = s0 + qq;
                        // lanes beyond the last sample re-read sample s (results discarded)
                        const int64_t lstride = (L > 1 && qq + 1 >= nq) ? 0 : p.sstride;
                        V x[NV][D], H[D][D], P[D][D], psi = V(T(0));
                        int bad = 0;
                        if constexpr (OP == OP_TANGENT) {
                            NhState<D, V> NS;
                            if constexpr (MODEL == MODEL_NH) {
                                V Hu[D][D];
                                gather<D, T, V, false>(p.u + (int64_t)s * p.sstride, lstride, nullptr, G, x);
                                grad_of<D, T, V>(G, x, Hu);
                                nh_state<D, V>(Hu, NS);
                                bad = n_bad(NS.x);
                            }
                            gather<D, T, V, MASKED>(p.v + (int64_t)s * p.sstride, lstride, p.mask, G, x);
                            grad_of<D, T, V>(G, x, H);
                            dstress<D, MODEL, T, V>(G, NS, H, P);
                        } else {
                            gather<D, T, V, false>(p.u + (int64_t)s * p.sstride, lstride, nullptr, G, x);
                            grad_of<D, T, V>(G, x, H);
                            stress<D, MODEL, T, V, HAS_PSI>(G, H, P, psi, bad);
                        }
                        if (MODEL == MODEL_NH && bad) {
                            n_inv += bad;
                            first_inv = min(first_inv, e);
                        }
                        if (HAS_PSI) {
#pragma unroll
                            for (int k = 0; k < L; ++k) {
                                if (qq + k >= nq) break;
                                const T w = pfem::lane(psi, k);
                                if (!isfinite(w)) ++n_nonfin;
                                wacc[qq + k] += w;
                                if (p.W_e) p.W_e[(int64_t)(s + k) * p.E + e] = w;
                            }
                        }
                        if (HAS_FORCE) {
                            V f[NV][D];
                            forces<D, T, V>(G, P, f);
#pragma unroll
                            for (int a = 0; a < NV; ++a)
#pragma unroll
                                for (int i = 0; i < D; ++i)
                                    *reinterpret_cast<V*>(fbuf + (((size_t)a * EB + el) * D + i) * ST + qq) = f[a][i];
                            if (!HAS_PSI && !isfinite(pfem::lane(f[0][0], 0))) ++n_nonfin;
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < ST; ++q) wsum[q] += (double)wacc[q];   // per-thread, fixed order
                if ((HAS_FORCE || p.f_ext) && !(p.dbg & 2)) {
                    bar_main(NT);
                    // ---------------- phase 2: block-local CSR gather, thread per occurrence
                    for (int oi = tid; oi < no; oi += NT) {
                        const int o = o0 + oi;
                        const int word = socc[oi];
                        const int node = word & OCC_NODE_MASK;
                        if (HAS_FORCE) {
                            A2 acc[SD / LA];
#pragma unroll
                            for (int k = 0; k < SD / LA; ++k) acc[k] = A2(T(0));
                            const int k1 = soe[oi + 1];
                            for (int k = soe[oi]; k < k1; ++k) {
                                const int j = sle[k];
                                const int el = j / NV, a = j - el * NV;
                                A2 f[SD / LA];
                                sld<T, SD>(fbuf + ((size_t)a * EB + el) * SD, reinterpret_cast<T*>(f));
#pragma unroll
                                for (int c = 0; c < SD / LA; ++c) acc[c] += f[c];
                            }
                            const T* accs = reinterpret_cast<const T*>(acc);
                            if (word & (OCC_NONOWNER | OCC_EARLIER)) {
                                // segment of a node finished elsewhere: partial[o][s][i]
#pragma unroll
                                for (int q = 0; q < ST; ++q) {
                                    if (q >= nq) break;
                                    T* dst = p.partial + ((int64_t)o * S + s0 + q) * D;
#pragma unroll
                                    for (int i = 0; i < D; ++i) dst[i] = accs[i * ST + q];
                                }
                            } else {
#pragma unroll
                                for (int q = 0; q < ST; ++q) {
                                    if (q >= nq) break;
                                    const int64_t nb = (int64_t)(s0 + q) * p.sstride + (int64_t)node * D;
#pragma unroll
                                    for (int i = 0; i < D; ++i) {
                                        T val = accs[i * ST + q];
                                        if (OP == OP_TANGENT && MASKED && __ldg(p.mask + (int64_t)node * D + i))
                                            val = __ldg(p.v + nb + i);
                                        p.out[nb + i] = val;
                                        if (cgdot) dot_acc += (double)__ldg(p.v + nb + i) * (double)val;
                                    }
                                }
                            }
                        }
                        if (HAS_PSI && p.f_ext && !(word & OCC_NONOWNER)) {
#pragma unroll
                            for (int q = 0; q < ST; ++q) {
                                if (q >= nq) break;
                                const int64_t nb = (int64_t)(s0 + q) * p.sstride + (int64_t)node * D;
                                double w = 0.0;
#pragma unroll
                                for (int i = 0; i < D; ++i)
                                    w += (double)__ldg(p.f_ext + (int64_t)node * D + i) * (double)__ldg(p.u + nb + i);
                                fsum[q] += w;
                            }
                        }
                    }
                }
                if (HAS_PSI && S > ST) {
                    // several chunks: flush this chunk's sums (per-sample channels)
                    bar_main(NT);
#pragma unroll
                    for (int q = 0; q < ST; ++q) {
                        double a = warp_sum(q < nq ? wsum[q] : 0.0), f2 = warp_sum(q < nq ? fsum[q] : 0.0);
                        if (lane == 0) { s_red[warp][q] = a; s_red[warp][ST + q] = f2; }
                        wsum[q] = fsum[q] = 0.0;
                    }
                    bar_main(NT);
                    if (tid < 2 * nq) {
                        const int q = tid % nq, kind = tid / nq;
                        double r = 0.0;
                        for (int w = 0; w < NT / 32; ++w) r += s_red[w][kind * ST + q];
                        p.blk_sum[(int64_t)(kind * S + s0 + q) * p.n_blocks + b] = r;
                    }
                } else if (HAS_FORCE && s0 + ST < S) {
                    bar_main(NT);   // fbuf is reused by the next chunk
                }
            }
            // ---------------- per-warp sums into shared memory (single-chunk case), CG dot
            const bool sums = ((HAS_PSI && S <= ST) || cgdot) && !(p.dbg & 8);
            if (sums) {
                if (HAS_PSI && S <= ST) {
#pragma unroll
                    for (int q = 0; q < ST; ++q) {
                        if (q >= S) break;
                        const double a = (double)warp_sum_t<T>((T)wsum[q]);
                        const double f2 = p.f_ext ? warp_sum(fsum[q]) : 0.0;
                        if (lane == 0) { s_red[warp][q] = a; s_red[warp][ST + q] = f2; }
                    }
                }
                if (cgdot) {
                    const double d2 = warp_sum(dot_acc);
                    if (lane == 0) s_red[warp][2 * ST] = d2;
                }
            }
            if (tid == 0) s_tk[it & 1] = req;    // the ticket after next (requested long ago)
            bar_main(NT);                        // phase-2 writes, s_red and s_tk complete
            // ---------------- warp 0: block sums, publish, chunk arrival; others go on
            if (warp == 0) {
                if (sums) {
                    if (HAS_PSI && S <= ST && lane < 2 * S) {
                        const int q = lane % S, kind = lane / S;
                        double r = 0.0;
                        for (int w = 0; w < NT / 32; ++w) r += s_red[w][kind * ST + q];
                        p.blk_sum[(int64_t)(kind * S + q) * p.n_blocks + b] = r;
                    }
                    if (cgdot && lane == 31) {
                        double r = 0.0;
                        for (int w = 0; w < NT / 32; ++w) r += s_red[w][2 * ST];
                        p.blk_sum[(int64_t)(2 * S) * p.n_blocks + b] = r;
                    }
                    __syncwarp();
                }
                int last = 0;
                if (lane == 0) {
                    // release is cumulative over the CTA's writes observed through the barrier
                    if (HAS_FORCE) st_release_gpu(p.flag + b, epoch + 1);
                    if ((HAS_PSI || cgdot) && !(p.dbg & 8)) {
                        const int ch = __ldg(p.blk_chunk + b);
                        const int need = arrivals * (__ldg(p.chunk_blk + ch + 1) - __ldg(p.chunk_blk + ch));
                        last = atom_add_acq_rel(p.chunk_done + ch, 1) == need - 1;
                    }
                }
                last = __shfl_sync(0xffffffffu, last, 0);
                if (last) {
                    const int ch = __ldg(p.blk_chunk + b);
                    bool dummy;
                    chunk_reduce<T>(p, ch, HAS_PSI ? 0 : 2 * S, cgdot ? 2 * S + 1 : 2 * S, 0, 1, lane, dummy);
                    int fin = 0;
                    if (lane == 0) {
                        p.chunk_done[ch] = 0;
                        fin = atom_add_acq_rel(&p.ctr->done, 1) == p.n_chunks - 1;
                    }
                    fin = __shfl_sync(0xffffffffu, fin, 0);
                    if (fin) finalize<T, HAS_PSI, OP == OP_TANGENT>(p, 0, 1, lane);
                }
            }
            t = t_next;
            t_next = s_tk[it & 1];
            ++it;
        }
        cp_wait<0>();
        if (t_next < p.n_blocks) { /* unreachable: t_next >= t */ }
    }

done:
    // every CTA reports its (rare) flag counts; the last CTA to leave publishes them and
    // resets the workspace counters for the next launch
    if (n_inv) {
        atomicAdd(&p.ctr->n_inv, n_inv);
        atomicMax(&p.ctr->first_inv, INT32_MAX - first_inv);
    }
    if (n_nonfin) atomicAdd(&p.ctr->n_nonfinite, n_nonfin);
    __threadfence();
    __syncthreads();
    if (tid == 0 && atomicAdd(&p.ctr->exit_count, 1) == (int)gridDim.x - 1) {
        __threadfence();
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
        p.ctr->fix_ticket = 0;
        p.ctr->exit_count = 0;
        __threadfence();
        p.ctr->epoch = epoch + 1;
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
        int bad = 0;
        if constexpr (OP == OP_TANGENT) {
            NhState<D, T> NS;
            if constexpr (MODEL == MODEL_NH) {
                T Hu[D][D];
                gather<D, T, T, false>(p.u + (int64_t)s * p.sstride, 0, nullptr, G, x);
                grad_of<D, T, T>(G, x, Hu);
                nh_state<D, T>(Hu, NS);
                bad = n_bad(NS.x);
            }
            gather<D, T, T, MASKED>(p.v + (int64_t)s * p.sstride, 0, p.mask, G, x);
            grad_of<D, T, T>(G, x, H);
            dstress<D, MODEL, T, T>(G, NS, H, P);
        } else {
            gather<D, T, T, false>(p.u + (int64_t)s * p.sstride, 0, nullptr, G, x);
            grad_of<D, T, T>(G, x, H);
            stress<D, MODEL, T, T, true>(G, H, P, psi, bad);
        }
        if (MODEL == MODEL_NH && bad) n_inv += bad;
        if (HAS_PSI) {
            const T W = psi;   // V_e folded into the moduli
            if (!isfinite(W)) ++n_nonfin;
            wtmp[(int64_t)s * p.E + e] = W;
        }
        if (HAS_FORCE) {
            T f[NV][D];
            forces<D, T, T>(G, P, f);
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

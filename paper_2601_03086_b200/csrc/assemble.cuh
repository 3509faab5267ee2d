// assemble.cuh — the fused element kernels of the hot path (§8 rows a2-a6) and their
// deterministic CSR-mode assembly.
//
// The plan (prep.cu) cuts the elements into blocks of at most EB consecutive plan positions,
// inside parts, and packs one record per block (RecLayout, common.cuh).
//
// Kernel A, staged form (k_assemble, several samples per call): a persistent grid of resident
// CTAs; CTA i takes blocks i, i+G, ... with no cross-CTA synchronisation.  Per block:
//   stage    one cp.async.bulk (TMA) copy of the block's record into shared memory, issued one
//            block ahead and completed on an mbarrier; the block's nodal fields (u, or v and the
//            NH state u for the tangent) copied into one shared buffer with cp.async
//   phase 1  thread per element: H, P / dP, psi; the d+1 nodal force vectors of all ST samples
//            -> fbuf[slot][element][dim][sample] (fp32 samples in FFMA2 pairs); W_e; per-warp
//            energy sums right after the element loop
//   phase 2  after one barrier (the next block's fields are then copied into the freed field
//            buffer): threads per node occurrence (fp32 four samples: one per component),
//            occurrences in descending entry count,
//            sum the block-local CSR entries in ascending (element, slot) order.  A node touched
//            only by this block gets its final value; otherwise the block writes its segment
//            seg[slot][s][d] (slots node-major, ascending block)
// Kernel A, direct form (assemble_direct.cuh, one sample per call): one CTA per block.
// Kernel B (k_node_finish): thread per multi-block node sums its segments in ascending block
// order (its CSR row segment by segment, reading R24), applies the mask and the CG p.q; per
// chunk and per part energy / f.u sums; the last CTA forms CG alpha, the flags and the
// pretraining loss.  Every floating-point sum has a fixed order: no float atomics anywhere
// (north star); results are independent of scheduling and bitwise reproducible.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "element.cuh"

namespace pfem {

enum { OP_ENERGY = 0, OP_ENERGY_RESIDUAL = 1, OP_RESIDUAL = 2, OP_TANGENT = 3 };
// staged kernel shape (measured): 256 threads, 2 resident CTAs per SM, T4 blocks of
// at most 256 elements (T3: 512)
constexpr int STAGED_MINB = 2;
constexpr int STAGED_NT = 256;
constexpr int EB3 = 256;
constexpr int ASM_NT = 256;   // main (element / occurrence) threads per CTA
constexpr int FIX_WARPS = 1;  // fix-up warps per CTA (+1 publisher warp)
constexpr int FIX_UNROLL = 4; // segments loaded together by one fix-up lane
constexpr int CHUNK = 32;     // blocks per reduction chunk (== CHUNK_BLOCKS of prep.cu)

template <int D>
struct EbOf {
    static constexpr int value = D == 3 ? EB3 : 512;   // compile-time block capacity
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
    const double* coords;  // [N][D] fp64 (on-the-fly geometry)
    int otf;               // form grad / vol from coords in the element pass (direct form)
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
    const int32_t* occ_seg;   // [n_occ] segment slot of a multi-block occurrence
    int n_fix;
    int n_seg_total;       // segments of multi-block nodes (bounds of occ_seg slots)
    int perm;              // plan positions are a permutation of the input elements
    RecLayout rec;
    uint32_t rec_base;     // staged kernel: record bytes [rec_base, rec_end) are copied
    uint32_t rec_end;      //   (RecLayout: conn / ent_pos / g .. loc_ent / end)
    const unsigned char* recs;
    // workspace
    Counters* ctr;
    double* blk_sum;       // [2S+2][n_blocks]: W_s, f.u_s, dot(main), dot(fix-up)
    double* chunk_sum;     // [2S+1][n_chunks]
    int32_t* part_cnt;     // [K] reduced chunks per part (0 at rest)
    T* partial;            // [n_occ][S][D]
    CgState* cg;           // non-null: fused p.q and alpha epilogue (S == 1)
    // pipelined CG (§8(f) row f3): the direct form stages p_new = z + beta p_old (z = D^-1 r or r,
    // the k_cg_dir formula) instead of copying v, and the node's owner occurrence stores p_new
    // into `v` (the p buffer of this iteration); p_old is the other buffer
    const T* cg_r;         // non-null: fused direction update
    const T* cg_pold;
    const T* cg_dinv;      // nullable (Jacobi)
    // pretraining-loss epilogue (§8(f) row f2), applied where the assembled value is written:
    // out = phi (.) (value - f_ext) * ep_scale; the last kernel-B CTA writes the batch-mean loss
    int ep;
    const T* ep_phi;       // nullable (1)
    T ep_scale;
    double* ep_loss;       // nullable
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

// ST per-lane values summed over the warp in one fixed shuffle tree: the first log2(ST)
// exchanges halve the values each lane carries (a lane keeps the half selected by its lane
// bit and adds its partner's copy of that half), the remaining ones are plain butterflies.
// Result q ends in lane q * (32 / ST).  (ST = 4: 6 shuffles instead of 20.)
template <class T, int ST>
__device__ __forceinline__ T warp_multi_sum(const T (&v)[ST], int lane) {
    static_assert(ST == 1 || ST == 2 || ST == 4, "ST");
    T c;
    if constexpr (ST == 4) {
        const bool h = lane & 16;
        T k0 = h ? v[2] : v[0], k1 = h ? v[3] : v[1];
        const T s0 = h ? v[0] : v[2], s1 = h ? v[1] : v[3];
        k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
        k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
        const bool h8 = lane & 8;
        c = (h8 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
    } else if constexpr (ST == 2) {
        const bool h = lane & 16;
        c = (h ? v[1] : v[0]) + __shfl_xor_sync(0xffffffffu, h ? v[0] : v[1], 16);
    } else {
        c = v[0];
    }
#pragma unroll
    for (int o = 32 / ST / 2; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    return c;
}

// fixed-order lane-strided sum of a[lo, hi): lane l adds a[lo+l], a[lo+l+32], ... in ascending
// order, the loads issued 8 at a time (a plain strided loop waits one latency per element)
__device__ __forceinline__ double lane_sum(const double* a, int lo, int hi, int lane) {
    double acc = 0.0;
    for (int c0 = lo + lane; c0 < hi; c0 += 32 * 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = c0 + 32 * u < hi ? __ldcg(a + c0 + 32 * u) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
    }
    return acc;
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

// the value written for DOF (node, i): the assembled sum, or the pretraining-loss gradient
template <class T>
__device__ __forceinline__ T out_value(const AsmParams<T>& p, int64_t dof, T val) {
    if (!p.ep) return val;
    const T fe = p.f_ext ? __ldg(p.f_ext + dof) : T(0);
    const T ph = p.ep_phi ? __ldg(p.ep_phi + dof) : T(1);
    return ph * (val - fe) * p.ep_scale;
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

// loads of n <= N contiguous values of the segment buffer (written by the previous grid,
// read-only here: the non-coherent path may cache them in L1, where the d components of
// neighbouring segments share sectors)
template <class T, int N>
__device__ __forceinline__ void ld_seg_vec(const T* p, T (&v)[N], int n) {
    if constexpr (sizeof(T) == 4 && N % 4 == 0) {
        if (n == N && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
            for (int k = 0; k < N / 4; ++k) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(p) + k);
                v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
            }
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = k < n ? __ldg(p + k) : T(0);
}

// stage block b: one bulk copy of its packed record (thread 0) + per-element material
// (cp.async, only for element-wise parameters); every thread commits one cp.async group
template <int D, class T, int NT>
__device__ __forceinline__ void stage_block(unsigned char* st, T* mst, uint64_t* bar, const AsmParams<T>& p, int b) {
    if (threadIdx.x == 0) {
        fence_proxy_async();   // earlier generic reads of this buffer precede the async write
        const uint32_t n = p.rec_end - p.rec_base;
        mbar_expect_tx(bar, n);
        tma_bulk_g2s(st, p.recs + (size_t)b * p.rec.bytes + p.rec_base, n, bar);
    }
}

// element-wise material of a block whose record has landed in shared memory: cp.async by
// input element id (the plan may visit elements in a locality order)
template <class T, int NT>
__device__ __forceinline__ void stage_material(T* mst, const unsigned char* rec, uint32_t base, const AsmParams<T>& p,
                                               int b) {
    const int32_t* eid = reinterpret_cast<const int32_t*>(rec + (p.rec.eid - base));   // present iff p.perm
    const int e0 = __ldg(p.blk_elem + b), ne = __ldg(p.blk_elem + b + 1) - e0;
    for (int el = threadIdx.x; el < ne; el += NT) {
        const int64_t e = p.perm ? eid[el] : e0 + el;
        if (p.mat.s0) cpn<sizeof(T)>(mst + el, p.mat.p0 + e * p.mat.s0);
        if (p.mat.s1) cpn<sizeof(T)>(mst + p.rec.eb + el, p.mat.p1 + e * p.mat.s1);
    }
}

// =====================================================================================
// Kernel A (CSR mode): persistent element-block kernel.  CTA i processes blocks i, i+G,
// i+2G, ... (no cross-CTA synchronisation at all).  Per block:
//   stage   : ONE TMA bulk copy of the block's packed record (conn, grad N, V, block-local
//             CSR, local vertex ids), prefetched one block ahead with mbarrier completion;
//             element-wise material and the block's nodal fields (u, v for the NH tangent)
//             prefetched into shared memory with cp.async (after the record has landed)
//   phase 1 : thread per element: H, P / dP, psi from shared memory only -> nodal forces of
//             all ST samples -> fbuf[slot][element][dim][sample] (fp32 pairs as FFMA2 lanes)
//   phase 2 : thread per node occurrence: sum its block-local CSR entries (ascending element,
//             slot).  Nodes touched only by this block: final value -> out.  Others: the
//             block's segment -> seg[o][s][d] (finished by kernel B).
// Kernel B: thread per multi-block node: out = sum of its segments in ascending block order
// (i.e. its CSR row summed segment by segment), masked rows, the CG dot; per-part energy
// totals and CG alpha by the last CTA.  Every sum has a fixed order: no float atomics.
// =====================================================================================
// staged nodal values of the element's vertices (ust[occ][D][ST]); pairs of fp32 samples
// are adjacent, so an F2 lane pair is one 8-byte shared load
template <int D, class T, class V, int ST>
__device__ __forceinline__ void load_staged_field(const T* __restrict__ ust, const int (&lv)[D + 1], int qq,
                                                  V (&x)[D + 1][D]) {
#pragma unroll
    for (int a = 0; a <= D; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const T* src = ust + ((size_t)lv[a] * D + i) * ST + qq;
            if constexpr (sizeof(V) == 8 && sizeof(T) == 4) {
                const float2 q = *reinterpret_cast<const float2*>(src);
                x[a][i] = V(q.x, q.y);
            } else if constexpr (sizeof(V) == 16 && sizeof(T) == 4) {
                x[a][i] = *reinterpret_cast<const V*>(src);
            } else {
                x[a][i] = *src;
            }
        }
}

// accumulate SD contiguous shared-memory values into acc without taking the address of a
// register array (keeps acc in registers)
template <class T, int SD>
__device__ __forceinline__ void sacc(const T* __restrict__ src, T (&acc)[SD]) {
    if constexpr (sizeof(T) == 4 && SD % 4 == 0) {
#pragma unroll
        for (int c = 0; c < SD / 4; ++c) {
            const float4 q = reinterpret_cast<const float4*>(src)[c];
            F2 a0(acc[4 * c], acc[4 * c + 1]), a1(acc[4 * c + 2], acc[4 * c + 3]);
            a0 = a0 + F2(q.x, q.y);
            a1 = a1 + F2(q.z, q.w);
            acc[4 * c] = a0.v.x; acc[4 * c + 1] = a0.v.y; acc[4 * c + 2] = a1.v.x; acc[4 * c + 3] = a1.v.y;
        }
    } else if constexpr (sizeof(T) == 4 && SD % 2 == 0) {
#pragma unroll
        for (int c = 0; c < SD / 2; ++c) {
            const float2 q = reinterpret_cast<const float2*>(src)[c];
            F2 a0(acc[2 * c], acc[2 * c + 1]);
            a0 = a0 + F2(q.x, q.y);
            acc[2 * c] = a0.v.x; acc[2 * c + 1] = a0.v.y;
        }
    } else if constexpr (sizeof(T) == 8 && SD % 2 == 0) {
#pragma unroll
        for (int c = 0; c < SD / 2; ++c) {
            const double2 q = reinterpret_cast<const double2*>(src)[c];
            acc[2 * c] += q.x;
            acc[2 * c + 1] += q.y;
        }
    } else {
#pragma unroll
        for (int c = 0; c < SD; ++c) acc[c] += src[c];
    }
}

// acc += b elementwise (registers; fp32 pairs as FADD2)
template <class T, int SD>
__device__ __forceinline__ void sacc_reg(const T (&b)[SD], T (&acc)[SD]) {
    if constexpr (sizeof(T) == 4 && SD % 2 == 0) {
#pragma unroll
        for (int c = 0; c < SD / 2; ++c) {
            F2 a0(acc[2 * c], acc[2 * c + 1]);
            a0 = a0 + F2(b[2 * c], b[2 * c + 1]);
            acc[2 * c] = a0.v.x; acc[2 * c + 1] = a0.v.y;
        }
    } else {
#pragma unroll
        for (int c = 0; c < SD; ++c) acc[c] += b[c];
    }
}

template <int D, class T, int NT, int ST, bool MASKED>
__device__ __forceinline__ void stage_fields(T* ust, const unsigned char* rec, uint32_t base, const T* src,
                                             const AsmParams<T>& p, int s0, int nq, int no) {
    // ust[occ][D][ST] <- src[s0 + q][node(occ)][i]; masked DOFs are zero-filled (src-size 0)
    // (rec holds the record from byte `base` on)
    const int32_t* socc = reinterpret_cast<const int32_t*>(rec + (p.rec.occ_node - base));
    for (int o = threadIdx.x; o < no; o += NT) {
        const int node = socc[o] & OCC_NODE_MASK;
        T* dst = ust + (size_t)o * D * ST;
        const T* g = src + (int64_t)s0 * p.sstride + (int64_t)node * D;
        uint32_t keep[D];
#pragma unroll
        for (int i = 0; i < D; ++i) keep[i] = MASKED ? (__ldg(p.mask + (int64_t)node * D + i) ? 0u : (uint32_t)sizeof(T)) : (uint32_t)sizeof(T);
        const int64_t ss = p.sstride;
        const uint32_t d0 = smem_addr(dst);
        if (nq == ST) {   // a full chunk: straight-line copies
#pragma unroll
            for (int q = 0; q < ST; ++q)
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    if (MASKED)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d0 + (uint32_t)((i * ST + q) * sizeof(T))),
                                     "l"(g + q * ss + i), "n"(sizeof(T)), "r"(keep[i]));
                    else
                        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d0 + (uint32_t)((i * ST + q) * sizeof(T))),
                                     "l"(g + q * ss + i), "n"(sizeof(T)));
                }
        } else {
            for (int q = 0; q < nq; ++q) {
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    if (MASKED)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_addr(dst + i * ST + q)),
                                     "l"(g + i), "n"(sizeof(T)), "r"(keep[i]));
                    else
                        cpn<sizeof(T)>(dst + i * ST + q, g + i);
                }
                g += ss;
            }
        }
        // a ragged last chunk: the unused sample lanes are zero (the four-sample lockstep
        // arithmetic then sees F = I there: finite, no inversion, nothing stored)
        for (int q = nq; q < ST; ++q)
#pragma unroll
            for (int i = 0; i < D; ++i) dst[i * ST + q] = T(0);
    }
}

// FEXT: the call passes f_ext (Pi = W - f.u; the pretraining epilogue); without it the f.u
// code is compiled out
template <int D, int MODEL, class T, int OP, int ST, bool MASKED, int EB, int NT, bool FEXT>
__global__ void __launch_bounds__(NT, STAGED_MINB)
k_assemble(const AsmParams<T> p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr bool HAS_FORCE = OP != OP_ENERGY;
    constexpr bool HAS_PSI = OP == OP_ENERGY || OP == OP_ENERGY_RESIDUAL;
    constexpr int NV = D + 1;
    constexpr int SD = ST * D;
    // staged fields (one buffer, refilled for the next block after phase 1): u (energy /
    // residual), v (linear tangent), v then u (NH tangent: the linearisation state)
    constexpr int NF = (OP == OP_TANGENT && MODEL == MODEL_NH) ? 2 : 1;
    // fp32 four-sample chunks: the element's samples in lockstep (F4 = two FFMA2 per operation;
    // measured: config 2 fp32 61.8 -> 55.9 us, config 3 K.v 154 -> 151 us, E+R unchanged)
    using V = std::conditional_t<(sizeof(T) == 4 && ST == 4), F4, std::conditional_t<(sizeof(T) == 4 && ST % 2 == 0), F2, T>>;
    constexpr int L = VTraits<V>::L;
    // fbuf[NV][EB][D][ST] in element order, gathered through loc_ent in phase 2
    constexpr bool P2DIM = sizeof(T) == 4 && ST == 4;   // phase 2: thread per (occurrence, component)
    const T* staged_src = (OP == OP_TANGENT) ? p.v : p.u;
    // shared layout: rec[2] | mat[2][2][EB] | ust[2][OCAP][D][ST] | fbuf[NV][EB][D][ST]
    const uint32_t srb = p.rec_end - p.rec_base;     // staged bytes of a record
    constexpr bool has_conn = false;   // every item stages its fields: no global gathers need node ids
    unsigned char* const stage0 = smem_raw;
    unsigned char* const stage1 = smem_raw + srb;
    T* mstage = reinterpret_cast<T*>(smem_raw + 2 * (size_t)srb);
    T* ustage = mstage + (((p.mat.s0 | p.mat.s1) != 0) ? 4 * EB : 0);   // material stage only if element-wise
    const size_t ust1 = (size_t)p.rec.ocap * D * ST;   // one staged field
    const size_t ust_sz = (size_t)NF * ust1;
    T* fbuf = ustage + ust_sz;
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ double s_red[2][NT / 32][2 * ST + 1];   // per-warp sums of an item, by item parity
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int S = p.S;
    // work items: (block, sample chunk of ST samples), chunk-major, so S > ST calls spread over
    // all CTAs; every item stages its chunk's nodal fields in shared memory
    constexpr bool pref = true;
    const int nb = p.n_blocks;
    const int NI = nb * ((S + ST - 1) / ST);
    // (CG products are single-sample calls: the direct forms carry the fused p.q)
    if (p.cg && ld_relaxed_i(&p.cg->done)) return;     // converged CG: the whole grid exits

    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    int n_inv = 0, first_inv = INT32_MAX, n_nonfin = 0;
    const LameScale<T> lsc = lame_scale<T>(p.mat);
    // uniform material: the Lame constants once per thread (the same arithmetic per element)
    const bool mat_uniform = p.mat.s0 == 0 && p.mat.s1 == 0;
    T mu_u = T(0), lam_u = T(0);
    if (mat_uniform) lame_elem<T>(p.mat, lsc, __ldg(p.mat.p0), __ldg(p.mat.p1), mu_u, lam_u);
    const int G = gridDim.x;
    int t = blockIdx.x;
    uint32_t par0 = 0u, par1 = 0u;   // mbarrier phase of each record buffer (registers, no arrays)
    // item t = (chunk c, block b), t = c nb + b, advanced by G without divisions
    int b = t, c = 0;
    while (b >= nb) { b -= nb; ++c; }
    int bn = b + G, cn = c;
    while (bn >= nb) { bn -= nb; ++cn; }
    // block metadata of the current item (the next item's is loaded one item ahead)
    int e0 = 0, ne = 0, no = 0;
    int b_prev = -1, s0_prev = 0, nq_prev = 1, cur_prev = 0;   // the item whose sums warp 0 still has to add
    // prologue: record of the first block, then its fields
    const bool has_mat = (p.mat.s0 | p.mat.s1) != 0;
    if (t < NI) {
        e0 = __ldg(p.blk_elem + b);
        ne = __ldg(p.blk_elem + b + 1) - e0;
        no = __ldg(p.blk_occ + b + 1) - __ldg(p.blk_occ + b);
        const int s0t = c * ST;
        stage_block<D, T, NT>(stage0, mstage, &s_bar[0], p, b);
        mbar_wait(&s_bar[0], 0);
        stage_fields<D, T, NT, ST, MASKED>(ustage, stage0, p.rec_base, staged_src, p, s0t, min(ST, S - s0t), no);
        if (NF == 2) stage_fields<D, T, NT, ST, false>(ustage + ust1, stage0, p.rec_base, p.u, p, s0t, min(ST, S - s0t), no);
        if (has_mat) stage_material<T, NT>(mstage, stage0, p.rec_base, p, b);
        cp_commit();
    }
    for (int it = 0; t < NI; ++it, t += G) {
        const int cur = it & 1;
        const int tn = t + G;
        const int s0 = c * ST;                 // this item's sample chunk
        const int nq = min(ST, S - s0);
        // the next item's block metadata, raw: the differences are formed after phase 1, where
        // they are first used, so no warp waits on these loads here (the early subtraction
        // held 6% of the kernel's stall samples, ncu r02b)
        int e0n = 0, e1n = 0, o0n = 0, o1n = 0;
        if (tn < NI) {
            e0n = __ldg(p.blk_elem + bn);
            e1n = __ldg(p.blk_elem + bn + 1);
            o0n = __ldg(p.blk_occ + bn);
            o1n = __ldg(p.blk_occ + bn + 1);
        }
        unsigned char* const sg_cur = cur ? stage1 : stage0;
        unsigned char* const sg_nxt = cur ? stage0 : stage1;
        mbar_wait(&s_bar[cur], cur ? par1 : par0);   // this block's record
        if (cur) par1 ^= 1u; else par0 ^= 1u;
        cp_wait<0>();                          // this thread's material + field copies of block b
        // One barrier covers the start of an item: everyone's field copies have landed, and
        // every thread has left the previous item's phase 2 (its record buffer, the force
        // buffer and the other half of s_red are free).  There is no barrier at an item's end.
        bar_main(NT);
        // prefetch the next item's record into the buffer the previous item used (its fields
        // follow after phase 1)
        if (tn < NI) stage_block<D, T, NT>(sg_nxt, mstage + 2 * EB * (cur ^ 1), &s_bar[cur ^ 1], p, bn);
        if (tid == 32 && tn + G < NI) {
            // the record after next into L2, so next iteration's bulk copy is an L2 hit
            int bnn = bn + G;
            while (bnn >= nb) bnn -= nb;
            const size_t rb = p.rec.bytes, off = (size_t)bnn * rb + p.rec_base;
            const uintptr_t a0 = (uintptr_t)(p.recs + off), a1 = (uintptr_t)(p.recs + off + (p.rec_end - p.rec_base));
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0)) : "memory");
        }
        const unsigned char* sg = sg_cur - p.rec_base;   // record byte offsets apply from here
        const int32_t* sconn = reinterpret_cast<const int32_t*>(sg + p.rec.conn);   // valid iff rec_base <= conn
        const T* sgrad = reinterpret_cast<const T*>(sg + p.rec.g);
        const T* svol = reinterpret_cast<const T*>(sg + p.rec.vol);
        const int32_t* socc = reinterpret_cast<const int32_t*>(sg + p.rec.occ_node);
        const uint16_t* soe = reinterpret_cast<const uint16_t*>(sg + p.rec.occ_ent);
        const uint16_t* sle = reinterpret_cast<const uint16_t*>(sg + p.rec.loc_ent);
        const uint16_t* slc = reinterpret_cast<const uint16_t*>(sg + p.rec.lconn);
        const int32_t* sseg = reinterpret_cast<const int32_t*>(sg + p.rec.occ_seg);
        const int32_t* seid = reinterpret_cast<const int32_t*>(sg + p.rec.eid);
        const T* smat = mstage + 2 * EB * cur;
        const T* ust = ustage;
        // the previous item's per-block sums (its warps' sums are complete: the barrier above)
        if (HAS_PSI && it > 0 && warp == 0 && lane < 2 * nq_prev) {
            const int q = lane % nq_prev, kind = lane / nq_prev;
            double r = 0.0;
            for (int w = 0; w < NT / 32; ++w) r += s_red[cur ^ 1][w][kind * ST + q];
            p.blk_sum[(int64_t)(kind * S + s0_prev + q) * p.n_blocks + b_prev] = r;
        }
        double fsum[ST];
#pragma unroll
        for (int q = 0; q < ST; ++q) fsum[q] = 0.0;
        {
            // ---------------- phase 1: elements
            T wacc[ST];
#pragma unroll
            for (int q = 0; q < ST; ++q) wacc[q] = T(0);
            for (int el = tid; el < ne; el += NT) {
                const int e = p.perm ? seid[el] : e0 + el;   // input element id (W_e, flags)
                T* const wrow = (HAS_PSI && p.W_e) ? p.W_e + (int64_t)s0 * p.E + e : nullptr;   // W_e[s0][e]
                Geo<D, T> G_;
                if (has_conn) {   // node ids: only the global gathers use them
                    if constexpr (D == 3) {
                        const int4 cv = *reinterpret_cast<const int4*>(sconn + el * 4);
                        G_.v[0] = cv.x; G_.v[1] = cv.y; G_.v[2] = cv.z; G_.v[3] = cv.w;
                    } else {
#pragma unroll
                        for (int a = 0; a <= D; ++a) G_.v[a] = sconn[el * NV + a];
                    }
                } else {
#pragma unroll
                    for (int a = 0; a <= D; ++a) G_.v[a] = 0;
                }
#pragma unroll
                for (int a = 0; a < D; ++a)
#pragma unroll
                    for (int j = 0; j < D; ++j) G_.g[a][j] = sgrad[(a * D + j) * EB + el];
                G_.V = svol[el];
                if (mat_uniform) {
                    G_.mu = mu_u * G_.V;
                    G_.lam = lam_u * G_.V;
                } else {
                    const T m0 = p.mat.s0 ? smat[el] : __ldg(p.mat.p0);
                    const T m1 = p.mat.s1 ? smat[EB + el] : __ldg(p.mat.p1);
                    lame_elem<T>(p.mat, lsc, m0, m1, G_.mu, G_.lam);
                    G_.mu *= G_.V;
                    G_.lam *= G_.V;
                }
                int lv[NV];   // vertex -> staged occurrence
                if constexpr (D == 3) {
                    const uint2 c = *reinterpret_cast<const uint2*>(slc + el * NV);
                    lv[0] = c.x & 0xffff; lv[1] = c.x >> 16; lv[2] = c.y & 0xffff; lv[3] = c.y >> 16;
                } else {
#pragma unroll
                    for (int a = 0; a < NV; ++a) lv[a] = slc[el * NV + a];
                }
#pragma unroll
                for (int a = 0; a < NV; ++a) PFEM_DCHECK(lv[a] < no);
#pragma unroll
                for (int qq = 0; qq < ST; qq += L) {
                    if (qq >= nq) break;
                    const int s = s0 + qq;
                    const int64_t lstride = (L > 1 && qq + 1 >= nq) ? 0 : p.sstride;
                    V x[NV][D], H[D][D], P[D][D], psi = V(T(0));
                    int bad = 0;
                    if constexpr (OP == OP_TANGENT) {
                        NhState<D, V> NS;
                        if constexpr (MODEL == MODEL_NH) {
                            V Hu[D][D];
                            if (pref) load_staged_field<D, T, V, ST>(ust + ust1, lv, qq, x);
                            else gather<D, T, V, false>(p.u + (int64_t)s * p.sstride, lstride, nullptr, G_, x);
                            grad_of<D, T, V>(G_, x, Hu);
                            nh_state<D, V>(Hu, NS);
                            bad = n_bad(NS.x);
                        }
                        if (pref) load_staged_field<D, T, V, ST>(ust, lv, qq, x);
                        else gather<D, T, V, MASKED>(staged_src + (int64_t)s * p.sstride, lstride, p.mask, G_, x);
                        grad_of<D, T, V>(G_, x, H);
                        dstress<D, MODEL, T, V>(G_, NS, H, P);
                    } else {
                        if (pref) load_staged_field<D, T, V, ST>(ust, lv, qq, x);
                        else gather<D, T, V, false>(staged_src + (int64_t)s * p.sstride, lstride, nullptr, G_, x);
                        grad_of<D, T, V>(G_, x, H);
                        stress<D, MODEL, T, V, HAS_PSI>(G_, H, P, psi, bad);
                    }
                    if (MODEL == MODEL_NH && bad) {
                        n_inv += bad;
                        first_inv = min(first_inv, e);
                    }
                    if (HAS_PSI) {
                        // non-finite check once per pair: w - w is 0 for finite w, NaN otherwise
                        if constexpr (L == 2) {
                            const V z = psi - psi;
                            if (!(z.v.x + z.v.y == 0.0f)) n_nonfin += (!isfinite(psi.v.x)) + (qq + 1 < nq && !isfinite(psi.v.y));
                        } else if constexpr (L == 4) {
                            const V z = psi - psi;
                            if (!((z.a.v.x + z.a.v.y) + (z.b.v.x + z.b.v.y) == 0.0f))
#pragma unroll
                                for (int k = 0; k < 4; ++k) n_nonfin += (qq + k < nq && !isfinite(pfem::lane(psi, k)));
                        }
#pragma unroll
                        for (int k = 0; k < L; ++k) {
                            if (qq + k >= nq) break;
                            const T w = pfem::lane(psi, k);
                            if (L == 1 && !isfinite(w)) ++n_nonfin;
                            wacc[qq + k] += w;
                            if (wrow) wrow[(int64_t)(qq + k) * p.E] = w;
                        }
                    }
                    if (HAS_FORCE) {
                        V f[NV][D];
                        forces<D, T, V>(G_, P, f);
#pragma unroll
                        for (int a = 0; a < NV; ++a)
#pragma unroll
                            for (int i = 0; i < D; ++i)
                                *reinterpret_cast<V*>(fbuf + ((size_t)(a * EB + el) * D + i) * ST + qq) = f[a][i];
                        if (!HAS_PSI && !isfinite(pfem::lane(f[0][0], 0))) ++n_nonfin;
                    }
                }
            }
            if (HAS_PSI) {
                // per-warp energy sums now, while other warps finish phase 1 (this half of s_red
                // was last read by warp 0 before the previous item's first barrier)
                T wv[ST];
#pragma unroll
                for (int q = 0; q < ST; ++q) wv[q] = q < nq ? wacc[q] : T(0);
                const T r = warp_multi_sum<T, ST>(wv, lane);
                if ((lane & (32 / ST - 1)) == 0) s_red[cur][warp][lane / (32 / ST)] = (double)r;
            }
            // the next block's fields, into the same buffer once every thread's phase-1 reads
            // are done (the barrier before phase 2); its record has had phase 1 to land, and
            // the copies have phase 2 to complete
            const bool do_p2 = HAS_FORCE || FEXT;
            bar_main(NT);   // every thread's phase-1 reads of the field buffer are done
            {
                if (tn < NI) {
                    mbar_wait(&s_bar[cur ^ 1], cur ? par0 : par1);
                    const int s0n = cn * ST, nqn = min(ST, S - s0n);
                    const int non = o1n - o0n;
                    stage_fields<D, T, NT, ST, MASKED>(ustage, sg_nxt, p.rec_base, staged_src, p, s0n, nqn, non);
                    if (NF == 2) stage_fields<D, T, NT, ST, false>(ustage + ust1, sg_nxt, p.rec_base, p.u, p, s0n, nqn, non);
                    if (has_mat)
                        stage_material<T, NT>(mstage + 2 * EB * (cur ^ 1), sg_nxt, p.rec_base, p, bn);
                }
                cp_commit();
            }
            if (do_p2) {
                // ---------------- phase 2: block-local CSR gather, occurrences in descending
                // entry count (occ_perm), entries in ascending (element, slot) order
                const uint16_t* sop = reinterpret_cast<const uint16_t*>(sg + p.rec.occ_perm);
                if constexpr (P2DIM) {
                    // fp32, four samples: one thread per (occurrence, component) sums the four
                    // samples of its component with one 16-byte load per entry.  The D threads
                    // of an occurrence read the D consecutive 16-byte granules of a force row,
                    // so a warp's gather spreads over the banks (the sample-pair split read the
                    // same granule from two lanes: 5.5 wavefronts per LDS.64 against 1.9 ideal,
                    // and phase 2 ran at the shared-memory pipe's limit; ncu r02b)
                    for (int w = tid; w < D * no; w += NT) {
                        const int o = w / D, i = w - o * D;
                        const int oi = (int)sop[o];
                        PFEM_DCHECK(oi < no);
                        const int word = socc[oi];
                        const int node = word & OCC_NODE_MASK;
                        if (HAS_FORCE) {
                            F2 a0(0.0f, 0.0f), a1(0.0f, 0.0f);   // samples (0, 1) and (2, 3)
                            const int kb = soe[oi], k1 = soe[oi + 1];
                            PFEM_DCHECK(kb <= k1 && k1 <= NV * ne);
                            const T* fb = fbuf + i * ST;
                            int k = kb;
                            for (; k + 1 < k1; k += 2) {   // ascending entry order, two gathers in flight
                                const int j0 = sle[k], j1 = sle[k + 1];
                                PFEM_DCHECK(j0 % EB < ne && j1 % EB < ne && j0 < NV * EB && j1 < NV * EB);
                                const float4 x0 = *reinterpret_cast<const float4*>(fb + (size_t)j0 * SD);
                                const float4 x1 = *reinterpret_cast<const float4*>(fb + (size_t)j1 * SD);
                                a0 = (a0 + F2(x0.x, x0.y)) + F2(x1.x, x1.y);
                                a1 = (a1 + F2(x0.z, x0.w)) + F2(x1.z, x1.w);
                            }
                            if (k < k1) {
                                const float4 x0 = *reinterpret_cast<const float4*>(fb + (size_t)sle[k] * SD);
                                a0 = a0 + F2(x0.x, x0.y);
                                a1 = a1 + F2(x0.z, x0.w);
                            }
                            const T acc4[4] = {a0.v.x, a0.v.y, a1.v.x, a1.v.y};
                            if (word & (OCC_NONOWNER | OCC_EARLIER)) {
                                const int slot = sseg[oi];
                                PFEM_DCHECK(slot >= 0 && slot < p.n_seg_total);
                                T* dst = p.partial + ((int64_t)slot * S + s0) * D + i;
#pragma unroll
                                for (int q = 0; q < ST; ++q) {
                                    if (q >= nq) break;
                                    dst[q * D] = acc4[q];
                                }
                            } else {
                                const int64_t dof = (int64_t)node * D + i;
                                const bool fixed = OP == OP_TANGENT && MASKED && __ldg(p.mask + dof);
#pragma unroll
                                for (int q = 0; q < ST; ++q) {
                                    if (q >= nq) break;
                                    const int64_t at = (int64_t)(s0 + q) * p.sstride + dof;
                                    const T val = fixed ? __ldg(p.v + at) : acc4[q];
                                    p.out[at] = out_value(p, dof, val);
                                }
                            }
                        }
                        if (HAS_PSI && FEXT && !(word & OCC_NONOWNER)) {
                            const int64_t dof = (int64_t)node * D + i;
                            const double fe = (double)__ldg(p.f_ext + dof);
#pragma unroll
                            for (int q = 0; q < ST; ++q) {
                                if (q >= nq) break;
                                fsum[q] += fe * (double)__ldg(p.u + (int64_t)(s0 + q) * p.sstride + dof);
                            }
                        }
                    }
                } else
                for (int w = tid; w < no; w += NT) {
                    // other chunk shapes (fp64 pairs, single samples): a thread per occurrence
                    const int oi = (int)sop[w];
                    PFEM_DCHECK(oi < no);
                    const int word = socc[oi];
                    const int node = word & OCC_NODE_MASK;
                    if (HAS_FORCE) {
                        T accs[SD];   // [D][ST]
#pragma unroll
                        for (int k = 0; k < SD; ++k) accs[k] = T(0);
                        const int kb = soe[oi], k1 = soe[oi + 1];
                        PFEM_DCHECK(kb <= k1 && k1 <= NV * ne);
                        for (int k = kb; k < k1; ++k) sacc<T, SD>(fbuf + (size_t)sle[k] * SD, accs);
                        if (word & (OCC_NONOWNER | OCC_EARLIER)) {
                            // this block's segment of a multi-block node: seg[slot][s][d], slots
                            // node-major (a node's segments contiguous, ascending block)
                            const int slot = sseg[oi];
                            PFEM_DCHECK(slot >= 0 && slot < p.n_seg_total);
#pragma unroll
                            for (int q = 0; q < ST; ++q) {
                                if (q >= nq) break;
                                T* dst = p.partial + ((int64_t)slot * S + s0 + q) * D;
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
                                    p.out[nb + i] = out_value(p, (int64_t)node * D + i, val);
                                }
                            }
                        }
                    }
                    if (HAS_PSI && FEXT && !(word & OCC_NONOWNER)) {
#pragma unroll
                        for (int q = 0; q < ST; ++q) {   // (compile-time q: fsum stays in registers)
                            if (q >= nq) continue;
                            const int64_t nb = (int64_t)(s0 + q) * p.sstride + (int64_t)node * D;
                            double w2 = 0.0;
#pragma unroll
                            for (int i = 0; i < D; ++i)
                                w2 += (double)__ldg(p.f_ext + (int64_t)node * D + i) * (double)__ldg(p.u + nb + i);
                            fsum[q] += w2;
                        }
                    }
                }
            }
        }
        // ---------------- per-item sums (the item's samples): the f.u sums join the energy sums
        // in this item's half of s_red; warp 0 adds the warps' sums after the next barrier
        if (HAS_PSI) {
#pragma unroll
            for (int q = 0; q < ST; ++q) {
                if (q >= nq) break;
                const double f2 = FEXT ? warp_sum(fsum[q]) : 0.0;
                if (lane == 0) s_red[cur][warp][ST + q] = f2;
            }
        }
        b_prev = b; s0_prev = s0; nq_prev = nq; cur_prev = cur;
        b = bn; c = cn; e0 = e0n; ne = e1n - e0n; no = o1n - o0n;
        bn += G;
        while (bn >= nb) { bn -= nb; ++cn; }
    }
    cp_wait<0>();
    if (HAS_PSI && b_prev >= 0) {   // the last item's per-block sums
        __syncthreads();
        if (warp == 0 && lane < 2 * nq_prev) {
            const int q = lane % nq_prev, kind = lane / nq_prev;
            double r = 0.0;
            for (int w = 0; w < NT / 32; ++w) r += s_red[cur_prev][w][kind * ST + q];
            p.blk_sum[(int64_t)(kind * S + s0_prev + q) * p.n_blocks + b_prev] = r;
        }
    }
    if (n_inv) {
        atomicAdd(&p.ctr->n_inv, n_inv);
        atomicMax(&p.ctr->first_inv, INT32_MAX - first_inv);
    }
    if (n_nonfin) atomicAdd(&p.ctr->n_nonfinite, n_nonfin);
    // let kernel B's prologue start (programmatic dependent launch); its grid-dependency
    // wait still covers every write of this grid
    asm volatile("griddepcontrol.launch_dependents;");
}

// Kernel B: finish multi-block nodes, chunked energy / dot reductions, totals, CG alpha.
template <int D, class T, int ST, bool MASKED, int NTB>
__global__ void __launch_bounds__(NTB)
k_node_finish(const AsmParams<T> p, int op_psi, int n_items) {
    __shared__ double s_red[NTB / 32];
    __shared__ int s_last;
    constexpr int SD = ST * D;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int S = ST == 1 ? 1 : p.S;   // single-sample instantiations serve S = 1 only (dispatch_st)
    const bool cgdot = p.cg != nullptr;
    // the first item's plan metadata (not written by kernel A) loads before the wait, so its
    // latency overlaps kernel A's tail
    const int nsc = (S + ST - 1) / ST;
    const int item0 = blockIdx.x * NTB + tid;
    int node0 = 0, k00 = 0, k10 = 0;
    if (item0 < n_items) {
        const int f = item0 / nsc;
        node0 = __ldg(p.fix_node + f);
        k00 = __ldg(p.fix_src_ptr + f);
        k10 = __ldg(p.fix_src_ptr + f + 1);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");    // kernel A complete and visible
    if (p.cg && ld_relaxed_i(&p.cg->done)) return;
    double dot_acc = 0.0;
    // ---------------- multi-block nodes: item = (fix entry, sample chunk)
    for (int item = item0; item < n_items; item += gridDim.x * NTB) {
        const int f = item / nsc, s0 = (item - f * nsc) * ST;
        const int nq = min(ST, S - s0);
        const bool first = item == item0;
        const int node = first ? node0 : __ldg(p.fix_node + f);
        const int k0 = first ? k00 : __ldg(p.fix_src_ptr + f), k1 = first ? k10 : __ldg(p.fix_src_ptr + f + 1);
        PFEM_DCHECK(k0 < k1 && k1 <= p.n_seg_total && node >= 0 && node < p.N);
        // the node's segments are contiguous: seg[k][s][d], k in [k0, k1) (ascending block)
        T acc[SD];
        ld_seg_vec<T, SD>(p.partial + ((int64_t)k0 * S + s0) * D, acc, nq * D);
        for (int k = k0 + 1; k < k1; ++k) {
            T v[SD];
            ld_seg_vec<T, SD>(p.partial + ((int64_t)k * S + s0) * D, v, nq * D);
#pragma unroll
            for (int c = 0; c < SD; ++c) acc[c] += v[c];
        }
#pragma unroll
        for (int q = 0; q < ST; ++q) {
            if (q >= nq) break;
            const int64_t nb = (int64_t)(s0 + q) * p.sstride + (int64_t)node * D;
#pragma unroll
            for (int i = 0; i < D; ++i) {
                T val = acc[q * D + i];
                if (MASKED && __ldg(p.mask + (int64_t)node * D + i)) val = __ldg(p.v + nb + i);
                p.out[nb + i] = out_value(p, (int64_t)node * D + i, val);
                if (cgdot) dot_acc += (double)__ldg(p.v + nb + i) * (double)val;
            }
        }
    }
    // ---------------- chunk reductions of the per-block sums (one chunk per CTA)
    const int rb = op_psi ? 0 : 2 * S;
    const int re = cgdot ? 2 * S + 1 : (op_psi ? 2 * S : 2 * S);
    // The CTA completing the last chunk of a part forms that part's totals (parts finish in
    // parallel; fixed order: blocks within a chunk, chunks within the part)
    const bool part_totals = op_psi && p.totals;
    for (int ch = blockIdx.x; ch < p.n_chunks; ch += gridDim.x) {
        const int c0 = __ldg(p.chunk_blk + ch), c1 = __ldg(p.chunk_blk + ch + 1);
        for (int r = rb + warp; r < re; r += NTB / 32) {
            double v = (c0 + lane < c1) ? __ldcg(p.blk_sum + (int64_t)r * p.n_blocks + c0 + lane) : 0.0;
            v = warp_sum(v);
            if (lane == 0) p.chunk_sum[(int64_t)r * p.n_chunks + ch] = v;
        }
        if (!part_totals) continue;
        __syncthreads();
        if (tid == 0) {
            int lo = 0, hi = p.K - 1;   // part of chunk ch: last k with part_chunk[k] <= ch
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (__ldg(p.part_chunk + mid) <= ch) lo = mid;
                else hi = mid - 1;
            }
            const int cb = __ldg(p.part_chunk + lo), ce = __ldg(p.part_chunk + lo + 1);
            __threadfence();
            s_last = atomicAdd(p.part_cnt + lo, 1) == ce - cb - 1 ? lo : -1;
        }
        __syncthreads();
        const int k = s_last;
        if (k >= 0) {
            __threadfence();
            const int cb = __ldg(p.part_chunk + k), ce = __ldg(p.part_chunk + k + 1);
            for (int s = warp; s < S; s += NTB / 32) {
                const double wv = warp_sum(lane_sum(p.chunk_sum + (int64_t)s * p.n_chunks, cb, ce, lane));
                const double fv = warp_sum(lane_sum(p.chunk_sum + (int64_t)(S + s) * p.n_chunks, cb, ce, lane));
                if (lane == 0) p.totals[(int64_t)s * p.K + k] = (T)(wv - fv);
            }
            if (tid == 0) p.part_cnt[k] = 0;
        }
        __syncthreads();   // s_last reused
    }
    if (cgdot) {
        const double t = cta_sum<NTB>(dot_acc, s_red);
        if (tid == 0) p.blk_sum[(int64_t)(2 * S + 1) * p.n_blocks + blockIdx.x] = t;   // per-CTA dot
    }
    // ---------------- last CTA: totals per (sample, part), CG alpha, flags, reset
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        s_last = atomicAdd(&p.ctr->exit_count, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (part_totals) {   // parts without elements have no chunk: their totals are 0 (R23)
        for (int pair = tid; pair < S * p.K; pair += NTB) {
            const int s = pair / p.K, k = pair - s * p.K;
            if (__ldg(p.part_chunk + k) == __ldg(p.part_chunk + k + 1)) p.totals[(int64_t)s * p.K + k] = T(0);
        }
    }
    if (part_totals && p.ep_loss) {   // pretraining loss: batch mean of Pi over (s, k), row order
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int j = 0; j < S * p.K; ++j) t += (double)ld_relaxed(p.totals + j);
            *p.ep_loss = t / ((double)S * (double)p.K);
        }
    }
    if (cgdot && warp == 0) {
        const double pq = warp_sum(lane_sum(p.chunk_sum + (int64_t)(2 * S) * p.n_chunks, 0, p.n_chunks, lane)) +
                          warp_sum(lane_sum(p.blk_sum + (int64_t)(2 * S + 1) * p.n_blocks, 0, (int)gridDim.x, lane));
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
        p.ctr->exit_count = 0;
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

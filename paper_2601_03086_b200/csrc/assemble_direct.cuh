// assemble_direct.cuh — the CSR-mode element kernel, "direct" form: one CTA per element
// block (non-persistent grid), element data read from the block's packed record in global
// memory (prefetched into L2 about one wave ahead with cp.async.bulk.prefetch), the nodal
// fields of the block's node occurrences staged in shared memory with cp.async, and only
// the staged fields, the block's CSR entries and the force buffer in shared memory, so
// several CTAs share an SM and hide each other's latencies.
//
//   phase 1, thread per element: H, P / dP, psi from the staged fields -> nodal forces of
//     all ST samples -> fbuf[slot][element][dim][sample]; W_e; per-sample energy sums
//   phase 2, thread per node occurrence: sum its block-local CSR entries (ascending element,
//     slot).  Nodes touched only by this block: final value -> out.  Others: the block's
//     segment -> partial[slot] (node-major, ascending block).
//   kernel B (k_node_finish, assemble.cuh) then sums the segments and the reductions.
//
// (Measured alternative, not kept: finishing multi-block nodes inside this kernel by a
// last-arrival counter per node (acq_rel atomic after the segment write) and the chunk
// reductions by the last CTA of each chunk removes kernel B, but the extra serialized
// round trips at the end of every CTA made it 1.6x slower on config 4.)
#pragma once

#include "assemble.cuh"

namespace pfem {

// L2 prefetch of bytes [off, off + len) of an array of `total` bytes (16-byte granules,
// clamped inside the array); a hint only, no registers or shared memory
__device__ __forceinline__ void l2_prefetch(const void* base, size_t total, size_t off, size_t len) {
    // absolute 16-byte granules: the start rounds down (the granule holding an in-bounds
    // byte lies inside the 256-byte aligned allocation), the end rounds down
    size_t e = off + len;
    if (e > total) e = total;
    const uintptr_t a0 = ((uintptr_t)base + off) & ~uintptr_t(15);
    const uintptr_t a1 = ((uintptr_t)base + e) & ~uintptr_t(15);
    if (a1 <= a0) return;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0)) : "memory");
}

// prefetch block b's record (from its gradients on; conn is not read here) and its
// per-element moduli into L2 (issued by one thread)
template <class T, bool OTF>
__device__ __forceinline__ void prefetch_record(const AsmParams<T>& p, int b) {
    const size_t rb = (size_t)p.rec.bytes, total = rb * p.n_blocks;
    // the fields the direct kernel reads (RecLayout order): fp32 (ent_pos layout)
    // [ent_pos, loc_ent), fp64 (loc_ent gather) [g, end); conn is not read here; on-the-fly
    // geometry skips the gradients and volumes [g, eid)
    const size_t b0 = (size_t)b * rb;
    if (OTF) {
        if (sizeof(T) == 4) {
            l2_prefetch(p.recs, total, b0 + p.rec.ent_pos, p.rec.g - p.rec.ent_pos);
            l2_prefetch(p.recs, total, b0 + p.rec.eid, p.rec.loc_ent - p.rec.eid);
        } else {
            l2_prefetch(p.recs, total, b0 + p.rec.eid, rb - p.rec.eid);
        }
    } else if (sizeof(T) == 4) {
        l2_prefetch(p.recs, total, b0 + p.rec.ent_pos, p.rec.loc_ent - p.rec.ent_pos);
    } else {
        l2_prefetch(p.recs, total, b0 + p.rec.g, rb - p.rec.g);
    }
    const int e0 = __ldg(p.blk_elem + b), e1 = __ldg(p.blk_elem + b + 1);
    const size_t E = (size_t)p.E, ne = (size_t)(e1 - e0);
    if (p.perm) return;   // element-wise materials are gathered through the permutation

    if (p.mat.s0) l2_prefetch(p.mat.p0, E * sizeof(T), e0 * sizeof(T), ne * sizeof(T));
    if (p.mat.s1) l2_prefetch(p.mat.p1, E * sizeof(T), e0 * sizeof(T), ne * sizeof(T));
}

// resident CTAs the register budget aims at (measured): fp64 linear single-sample calls 4 per SM
// (64 registers; config 4 134.5 -> 132.4 us), several-sample fp32 calls 6
constexpr int DIRECT_MINB64 = 4;
constexpr int DIRECT_MINBS = 6;
// register budget (measured): fp32 single-sample calls 64 registers (8% faster on config 5
// than the default); several-sample fp32 calls 80; fp64 linear single-sample calls 64 (4 CTAs
// per SM with the 384-element blocks: config 4 134.5 -> 132.4 us); fp64 Neo-Hookean and fp64
// several-sample calls the compiler's own allocation (a 40-register cap spilled hundreds of
// bytes per thread)
template <int D, int MODEL, class T, int OP, int ST, bool MASKED, int NT, bool PERM, bool OTF>
__global__ void __launch_bounds__(NT, ST > 1 ? (sizeof(T) == 4 ? DIRECT_MINBS : 0)
                                            : (sizeof(T) == 4 ? 65536 / (NT * 64) : (MODEL == MODEL_LINEAR ? DIRECT_MINB64 : 0)))
k_assemble_direct(const AsmParams<T> p) {
    // shared: ust[NF][OCAP][D][ST] (staged nodal fields) | [le[(d+1) EB] u16] | fbuf
    // EPOS (fp32): fbuf[(d+1) EB entries][D][ST], element vertex forces scattered to their
    //   block-CSR entry (ent_pos), so phase 2 reads an occurrence's entries contiguously
    // !EPOS (fp64): fbuf[NV][EB][D][ST] written conflict-free by consecutive elements, phase 2
    //   gathers through loc_ent (le, copied to shared memory); fp64 vertex vectors are 24-byte
    //   and scattered 8-byte stores saturate the shared-memory pipe
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ double s_red[NT / 32][2 * ST + 1];
    constexpr bool HAS_FORCE = OP != OP_ENERGY;
    constexpr bool HAS_PSI = OP == OP_ENERGY || OP == OP_ENERGY_RESIDUAL;
    constexpr int NV = D + 1;
    constexpr int SD = ST * D;
    constexpr int NF = (OP == OP_TANGENT && MODEL == MODEL_NH) ? 2 : 1;   // NH tangent stages u and v
    using V = std::conditional_t<(sizeof(T) == 4 && ST % 2 == 0), F2, T>;
    constexpr int L = VTraits<V>::L;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // single-sample instantiations serve S = 1 only (dispatch_st); folding it into the fp64 code
    // measured faster (config 4 132.4 -> 130.5 us), into the fp32 code slower (config 5 71 -> 73)
    const int S = (ST == 1 && sizeof(T) == 8) ? 1 : p.S;
    const int EB = p.rec.eb;                                    // record / fbuf stride
    const size_t ust_sz = (size_t)p.rec.ocap * D * ST;
    T* ust = reinterpret_cast<T*>(smem_raw);
    constexpr bool EPOS = sizeof(T) == 4;
    uint16_t* le = reinterpret_cast<uint16_t*>(ust + NF * ust_sz);
    T* fbuf = reinterpret_cast<T*>(smem_raw + ((NF * ust_sz * sizeof(T) + (EPOS ? 0 : 2 * (size_t)NV * EB) + 15) &
                                               ~size_t(15)));
    // on-the-fly geometry: the vertex coordinates of the block's node occurrences [ocap][D]
    double* scoord = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(fbuf + (HAS_FORCE ? (size_t)ST * D * NV * EB : 0)) + 15) & ~uintptr_t(15));
    const bool cgdot = OP == OP_TANGENT && p.cg != nullptr;
    if (p.cg && ld_relaxed_i(&p.cg->done)) return;
    const int b = blockIdx.x;
    if (p.lag > 0 && tid == 0 && b + p.lag < p.n_blocks) prefetch_record<T, OTF>(p, b + p.lag);
    const unsigned char* rg = p.recs + (size_t)b * p.rec.bytes;
    const unsigned char* rgb = rg;   // the record is read from global memory (read-only path)
    const int e0 = __ldg(p.blk_elem + b), ne = __ldg(p.blk_elem + b + 1) - e0;
    const int no = __ldg(p.blk_occ + b + 1) - __ldg(p.blk_occ + b);
    const int32_t* socc = reinterpret_cast<const int32_t*>(rgb + p.rec.occ_node);
    const uint16_t* soe = reinterpret_cast<const uint16_t*>(rgb + p.rec.occ_ent);
    const int32_t* sseg = reinterpret_cast<const int32_t*>(rgb + p.rec.occ_seg);
    if (!EPOS && HAS_FORCE) {   // block-local CSR entries -> shared (async, lands by the first barrier)
        const int nchunk = (2 * NV * ne + 15) / 16;
        for (int c = tid; c < nchunk; c += NT) cpn<16>(le + 8 * c, rg + p.rec.loc_ent + 16 * c);
    }
    // this thread's first occurrence: phase-2 metadata loaded now, in flight during phase 1
    int w_0 = 0, kb_0 = 0, k1_0 = 0, sl_0 = -1;
    if ((HAS_FORCE || p.f_ext) && tid < no) {
        w_0 = __ldg(socc + tid);
        kb_0 = __ldg(soe + tid);
        k1_0 = __ldg(soe + tid + 1);
        sl_0 = __ldg(sseg + tid);
    }
    int n_inv = 0, first_inv = INT32_MAX, n_nonfin = 0;
    double dot_acc = 0.0;
    double wsum[ST], fsum[ST];
#pragma unroll
    for (int q = 0; q < ST; ++q) wsum[q] = fsum[q] = 0.0;
    // uniform-nu Lame constants: one thread forms them (two divisions), read after the barrier
    __shared__ T s_lame[2];
    LameScale<T> lsc;
    lsc.on = p.mat.kind != KIND_LAME && p.mat.s1 == 0;
    if (lsc.on && tid == 0) lame_of<T>(p.mat.kind, T(1), __ldg(p.mat.p1), s_lame[0], s_lame[1]);
    for (int s0 = 0; s0 < S; s0 += ST) {
        const int nq = min(ST, S - s0);
        if (OP == OP_TANGENT && ST == 1 && p.cg_r) {
            // pipelined CG: p_new = z + beta p_old formed while staging (k_cg_dir's formula, so
            // the iterates are those of the unfused loop); the owner occurrence stores p_new
            const int32_t* so = reinterpret_cast<const int32_t*>(rgb + p.rec.occ_node);
            const T beta = (T)p.cg->beta;
            T* pnew = const_cast<T*>(p.v);
            for (int o = tid; o < no; o += NT) {
                const int word = __ldg(so + o);
                const int64_t base = (int64_t)(word & OCC_NODE_MASK) * D;
                T pn[D];
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    const T rv = __ldg(p.cg_r + base + i);
                    const T z = p.cg_dinv ? __ldg(p.cg_dinv + base + i) * rv : rv;
                    pn[i] = fma(beta, __ldg(p.cg_pold + base + i), z);
                }
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    ust[o * D + i] = (MASKED && __ldg(p.mask + base + i)) ? T(0) : pn[i];
                    if (!(word & OCC_NONOWNER)) pnew[base + i] = pn[i];
                }
            }
            if (NF == 2) stage_fields<D, T, NT, ST, false>(ust + ust_sz, rgb, 0u, p.u, p, s0, nq, no);
        } else if (OP == OP_TANGENT) {
            stage_fields<D, T, NT, ST, MASKED>(ust, rgb, 0u, p.v, p, s0, nq, no);
            if (NF == 2) stage_fields<D, T, NT, ST, false>(ust + ust_sz, rgb, 0u, p.u, p, s0, nq, no);
        } else {
            stage_fields<D, T, NT, ST, false>(ust, rgb, 0u, p.u, p, s0, nq, no);
        }
        if (OTF && s0 == 0) {   // vertex coordinates (fp64) of the block's occurrences
            const int32_t* so = reinterpret_cast<const int32_t*>(rgb + p.rec.occ_node);
            for (int o = tid; o < no; o += NT) {
                const int node = __ldg(so + o) & OCC_NODE_MASK;
#pragma unroll
                for (int i = 0; i < D; ++i) cpn<8>(scoord + o * D + i, p.coords + (int64_t)node * D + i);
            }
        }
        cp_commit();
        T wacc[ST];
#pragma unroll
        for (int q = 0; q < ST; ++q) wacc[q] = T(0);
        cp_wait<0>();
        __syncthreads();     // staged fields, loc_ent and Lame constants visible
        lsc.mu1 = s_lame[0];
        lsc.lam1 = s_lame[1];
        // ---------------- phase 1: elements (one per thread and pass)
        for (int el = tid; el < ne; el += NT) {
            // input element id (W_e, material, flags): identity order needs no load, and the
            // material load then does not wait on the id
            const int e = PERM ? __ldg(reinterpret_cast<const int32_t*>(rgb + p.rec.eid) + el) : e0 + el;
            Geo<D, T> G;
            int lv[NV], ep[NV];   // vertex -> staged occurrence, vertex -> block-CSR entry
            if constexpr (D == 3) {
                const uint2 c = __ldg(reinterpret_cast<const uint2*>(rgb + p.rec.lconn) + el);
                lv[0] = c.x & 0xffff; lv[1] = c.x >> 16; lv[2] = c.y & 0xffff; lv[3] = c.y >> 16;
#pragma unroll
                for (int a = 0; a < NV; ++a) PFEM_DCHECK(lv[a] < no);
                if (EPOS) {
                    const uint2 q = __ldg(reinterpret_cast<const uint2*>(rgb + p.rec.ent_pos) + el);
                    ep[0] = q.x & 0xffff; ep[1] = q.x >> 16; ep[2] = q.y & 0xffff; ep[3] = q.y >> 16;
                }
            } else {
                const uint16_t* lc = reinterpret_cast<const uint16_t*>(rgb + p.rec.lconn) + el * NV;
                const uint16_t* lp = reinterpret_cast<const uint16_t*>(rgb + p.rec.ent_pos) + el * NV;
#pragma unroll
                for (int a = 0; a < NV; ++a) {
                    lv[a] = __ldg(lc + a);
                    if (EPOS) ep[a] = __ldg(lp + a);
                }
            }
            {
                if constexpr (OTF) {
                    // grad N_a and V_e formed in fp64 from the staged vertex coordinates (the
                    // formula of pfem_mesh_prepare), then rounded to T like the prepared arrays
                    double X[NV][D], inv[D][D];
#pragma unroll
                    for (int a = 0; a < NV; ++a)
#pragma unroll
                        for (int i = 0; i < D; ++i) X[a][i] = scoord[lv[a] * D + i];
                    const double det = geometry_of<D>(X, inv);
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int j = 0; j < D; ++j) G.g[a][j] = (T)inv[a][j];
                    G.V = (T)(fabs(det) / (D == 2 ? 2.0 : 6.0));
                } else {
                    const T* sg = reinterpret_cast<const T*>(rgb + p.rec.g);
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int j = 0; j < D; ++j) G.g[a][j] = __ldg(sg + (a * D + j) * EB + el);
                    G.V = __ldg(reinterpret_cast<const T*>(rgb + p.rec.vol) + el);
                }
                const T m0 = __ldg(p.mat.p0 + (int64_t)e * p.mat.s0);
                const T m1 = __ldg(p.mat.p1 + (int64_t)e * p.mat.s1);
                lame_elem<T>(p.mat, lsc, m0, m1, G.mu, G.lam);
                G.mu *= G.V;
                G.lam *= G.V;
            }
#pragma unroll
            for (int qq = 0; qq < ST; qq += L) {
                if (qq >= nq) break;
                const int s = s0 + qq;
                V x[NV][D], H[D][D], P[D][D], psi = V(T(0));
                int bad = 0;
                if constexpr (OP == OP_TANGENT) {
                    NhState<D, V> NS;
                    if constexpr (MODEL == MODEL_NH) {
                        V Hu[D][D];
                        load_staged_field<D, T, V, ST>(ust + ust_sz, lv, qq, x);
                        grad_of<D, T, V>(G, x, Hu);
                        nh_state<D, V>(Hu, NS);
                        bad = n_bad(NS.x);
                    }
                    load_staged_field<D, T, V, ST>(ust, lv, qq, x);
                    grad_of<D, T, V>(G, x, H);
                    dstress<D, MODEL, T, V>(G, NS, H, P);
                } else {
                    load_staged_field<D, T, V, ST>(ust, lv, qq, x);
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
                            *reinterpret_cast<V*>(fbuf + ((size_t)(EPOS ? ep[a] : a * EB + el) * D + i) * ST + qq) = f[a][i];
                    if (!HAS_PSI && !isfinite(pfem::lane(f[0][0], 0))) ++n_nonfin;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < ST; ++q) wsum[q] += (double)wacc[q];
        if (HAS_FORCE || p.f_ext) {
            __syncthreads();
            // ---------------- phase 2: block-local CSR gather, thread per occurrence
            for (int oi = tid; oi < no; oi += NT) {
                const bool first = oi == tid;
                const int word = first ? w_0 : __ldg(socc + oi);
                const int node = word & OCC_NODE_MASK;
                if (HAS_FORCE) {
                    T accs[SD];
#pragma unroll
                    for (int k = 0; k < SD; ++k) accs[k] = T(0);
                    const int k1 = first ? k1_0 : __ldg(soe + oi + 1);
                    for (int k = first ? kb_0 : __ldg(soe + oi); k < k1; ++k) {
                        const int slot = EPOS ? k : (int)le[k];   // (record loc_ent = force-buffer slot)
                        PFEM_DCHECK(slot < (D + 1) * EB && (EPOS || slot % EB < ne));
                        sacc<T, SD>(fbuf + (size_t)slot * SD, accs);
                    }
                    if (word & (OCC_NONOWNER | OCC_EARLIER)) {
                        const int slot = first ? sl_0 : __ldg(sseg + oi);
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
            __syncthreads();
#pragma unroll
            for (int q = 0; q < ST; ++q) {
                double a = warp_sum(q < nq ? wsum[q] : 0.0), f2 = warp_sum(q < nq ? fsum[q] : 0.0);
                if (lane == 0) { s_red[warp][q] = a; s_red[warp][ST + q] = f2; }
                wsum[q] = fsum[q] = 0.0;
            }
            __syncthreads();
            if (tid < 2 * nq) {
                const int q = tid % nq, kind = tid / nq;
                double r = 0.0;
                for (int w = 0; w < NT / 32; ++w) r += s_red[w][kind * ST + q];
                p.blk_sum[(int64_t)(kind * S + s0 + q) * p.n_blocks + b] = r;
            }
        }
        if (s0 + ST < S) __syncthreads();   // ust / fbuf reused by the next sample chunk
    }
    if ((HAS_PSI && S <= ST) || cgdot) {
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
        __syncthreads();
        if (warp == 0) {
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
        }
    }
    if (n_inv) {
        atomicAdd(&p.ctr->n_inv, n_inv);
        atomicMax(&p.ctr->first_inv, INT32_MAX - first_inv);
    }
    if (n_nonfin) atomicAdd(&p.ctr->n_nonfinite, n_nonfin);
    asm volatile("griddepcontrol.launch_dependents;");
}

}  // namespace pfem

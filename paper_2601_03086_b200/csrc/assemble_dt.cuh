// assemble_dt.cuh — the CSR-mode element kernel for single-sample calls, "in-place" form:
// one CTA per element block; the block's record is bulk-copied (TMA, two copies on one
// mbarrier) into shared memory at CTA start while the same CTA gathers the nodal fields of
// its node occurrences (node ids read from the record in global memory, cp.async), so the
// element-data stream and the field gather are in flight together, and phase 1 reads
// shared memory only.  The force buffer overwrites the element geometry it was formed from:
//
//   shared  [0, A)      record bytes [g, vol + EB s): rows 0 .. d^2 of [.][EB] T (grad N, V)
//           [A, A + X)  two more rows [EB] T: element-wise moduli (cp.async), then forces
//           [A + X, ..) record bytes [eid, end): eid, occurrences, lconn, segment slots, loc_ent
//           then the staged fields ust[NF][ocap][D]
//   fbuf    row k = a d + i (vertex a, component i), column el: row k of the layout above.
//           Thread el reads rows 0 .. d^2 (and the moduli rows) of column el before it
//           writes forces there, and no other thread touches column el, so the in-place
//           write needs no barrier; d (d+1) force rows = d^2 + 1 geometry rows + d - 1 more.
//
// Phase 2 (thread per occurrence) gathers the block-local CSR entries, slot = a EB + el
// (loc_ent), from the rows a d + i, in ascending (element, slot) order like every other
// CSR form, so the results are bitwise those of k_assemble_direct.  Kernel B is unchanged.
// (Compared with k_assemble_direct, which reads the element data from global memory after
// its field barrier, the per-CTA chain loses one dependent memory round trip, and the
// shared footprint stays ~50 KB for fp64 T4 blocks of 384: four CTAs per SM.)
#pragma once

#include "assemble_direct.cuh"

namespace pfem {

constexpr int DT_XROWS = 2;   // extra shared rows beyond the record's d^2 + 1 geometry rows

struct DtLayout {
    uint32_t a;      // bytes of record part 1 (g, vol) = (d^2 + 1) EB s
    uint32_t x;      // extra rows
    uint32_t b;      // bytes of record part 2 [eid, end)
    uint32_t ust;    // offset of the staged fields
    uint32_t total;
    bool ok;
};

// host + device: the in-place form needs the geometry rows contiguous and 16-byte granular
__host__ __device__ inline DtLayout dt_layout(const RecLayout& R, int D, int tsize, int nf) {
    DtLayout L;
    const uint32_t row = (uint32_t)R.eb * (uint32_t)tsize;
    L.ok = row % 16 == 0 && R.vol - R.g == (uint32_t)(D * D) * row && R.eid == R.vol + row;
    L.a = (uint32_t)(D * D + 1) * row;
    L.x = DT_XROWS * row;
    L.b = R.bytes - R.eid;
    L.ust = L.a + L.x + L.b;
    L.total = L.ust + (uint32_t)((nf * (size_t)R.ocap * D * tsize + 15) / 16 * 16);
    return L;
}

template <int D, int MODEL, class T, int OP, bool MASKED, int NT, bool PERM>
__global__ void __launch_bounds__(NT, sizeof(T) == 4 ? 65536 / (NT * 64) : (MODEL == MODEL_LINEAR ? DIRECT_MINB64 : 0))
k_assemble_dt(const AsmParams<T> p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ double s_red[NT / 32][3];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ T s_lame[2];
    constexpr bool HAS_FORCE = OP != OP_ENERGY;
    constexpr bool HAS_PSI = OP == OP_ENERGY || OP == OP_ENERGY_RESIDUAL;
    constexpr int NV = D + 1;
    constexpr int NF = (OP == OP_TANGENT && MODEL == MODEL_NH) ? 2 : 1;   // NH tangent stages u and v
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int EB = p.rec.eb;
    const DtLayout L = dt_layout(p.rec, D, (int)sizeof(T), NF);
    T* const fb = reinterpret_cast<T*>(smem_raw);                     // rows [.][EB]
    const unsigned char* const r2 = smem_raw + L.a + L.x - p.rec.eid;  // record offsets >= eid apply here
    T* const ust = reinterpret_cast<T*>(smem_raw + L.ust);
    const size_t ust_sz = (size_t)p.rec.ocap * D;
    const bool cgdot = OP == OP_TANGENT && p.cg != nullptr;
    if (p.cg && ld_relaxed_i(&p.cg->done)) return;
    const int b = blockIdx.x;
    const unsigned char* rg = p.recs + (size_t)b * p.rec.bytes;
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        mbar_fence_init();
        mbar_expect_tx(&s_bar, L.a + L.b);
        tma_bulk_g2s(smem_raw, rg + p.rec.g, L.a, &s_bar);
        tma_bulk_g2s(smem_raw + L.a + L.x, rg + p.rec.eid, L.b, &s_bar);
        // a later block's record into L2 (about one wave ahead), so its bulk copy hits L2
        if (p.lag > 0 && b + p.lag < p.n_blocks) {
            const size_t rb = (size_t)p.rec.bytes;
            l2_prefetch(p.recs, rb * p.n_blocks, (size_t)(b + p.lag) * rb + p.rec.g, rb - p.rec.g);
            if (!PERM) {
                const int f0 = __ldg(p.blk_elem + b + p.lag), f1 = __ldg(p.blk_elem + b + p.lag + 1);
                if (p.mat.s0 == 1) l2_prefetch(p.mat.p0, (size_t)p.E * sizeof(T), f0 * sizeof(T), (size_t)(f1 - f0) * sizeof(T));
                if (p.mat.s1 == 1) l2_prefetch(p.mat.p1, (size_t)p.E * sizeof(T), f0 * sizeof(T), (size_t)(f1 - f0) * sizeof(T));
            }
        }
    }
    const int e0 = __ldg(p.blk_elem + b), ne = __ldg(p.blk_elem + b + 1) - e0;
    const int no = __ldg(p.blk_occ + b + 1) - __ldg(p.blk_occ + b);
    // ---------------- stage: nodal fields (node ids from the record in global memory) and
    // element-wise moduli (input order only) into the extra rows, while the record lands
    if (OP == OP_TANGENT && p.cg_r) {
        // pipelined CG: p_new = z + beta p_old formed while staging (k_cg_dir's formula, so
        // the iterates are those of the unfused loop); the owner occurrence stores p_new
        const int32_t* so = reinterpret_cast<const int32_t*>(rg + p.rec.occ_node);
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
        if (NF == 2) stage_fields<D, T, NT, 1, false>(ust + ust_sz, rg, 0u, p.u, p, 0, 1, no);
    } else if (OP == OP_TANGENT) {
        stage_fields<D, T, NT, 1, MASKED>(ust, rg, 0u, p.v, p, 0, 1, no);
        if (NF == 2) stage_fields<D, T, NT, 1, false>(ust + ust_sz, rg, 0u, p.u, p, 0, 1, no);
    } else {
        stage_fields<D, T, NT, 1, false>(ust, rg, 0u, p.u, p, 0, 1, no);
    }
    T* const xm0 = fb + (size_t)(D * D + 1) * EB;   // moduli rows (element-wise, input order)
    T* const xm1 = xm0 + EB;
    if (!PERM) {
        for (int el = tid; el < ne; el += NT) {
            if (p.mat.s0) cpn<sizeof(T)>(xm0 + el, p.mat.p0 + (int64_t)(e0 + el) * p.mat.s0);
            if (p.mat.s1) cpn<sizeof(T)>(xm1 + el, p.mat.p1 + (int64_t)(e0 + el) * p.mat.s1);
        }
    }
    cp_commit();
    LameScale<T> lsc;
    lsc.on = p.mat.kind != KIND_LAME && p.mat.s1 == 0;
    if (lsc.on && tid == 0) lame_of<T>(p.mat.kind, T(1), __ldg(p.mat.p1), s_lame[0], s_lame[1]);
    const T m0u = p.mat.s0 ? T(0) : __ldg(p.mat.p0), m1u = p.mat.s1 ? T(0) : __ldg(p.mat.p1);
    int n_inv = 0, first_inv = INT32_MAX, n_nonfin = 0;
    cp_wait<0>();
    __syncthreads();          // fields, moduli, Lame constants and the mbarrier init visible
    mbar_wait(&s_bar, 0);     // the record has landed
    lsc.mu1 = s_lame[0];
    lsc.lam1 = s_lame[1];
    const int32_t* seid = reinterpret_cast<const int32_t*>(r2 + p.rec.eid);
    const int32_t* socc = reinterpret_cast<const int32_t*>(r2 + p.rec.occ_node);
    const uint16_t* soe = reinterpret_cast<const uint16_t*>(r2 + p.rec.occ_ent);
    const uint16_t* slc = reinterpret_cast<const uint16_t*>(r2 + p.rec.lconn);
    const int32_t* sseg = reinterpret_cast<const int32_t*>(r2 + p.rec.occ_seg);
    const uint16_t* sle = reinterpret_cast<const uint16_t*>(r2 + p.rec.loc_ent);
    T wacc = T(0);
    // ---------------- phase 1: elements (thread el; shared memory only, forces in place)
    for (int el = tid; el < ne; el += NT) {
        const int e = PERM ? seid[el] : e0 + el;   // input element id (W_e, moduli, flags)
        Geo<D, T> G;
        int lv[NV];
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
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int j = 0; j < D; ++j) G.g[a][j] = fb[(a * D + j) * EB + el];
        G.V = fb[D * D * EB + el];
        {
            T m0, m1;
            if (PERM) {
                m0 = p.mat.s0 ? __ldg(p.mat.p0 + (int64_t)e * p.mat.s0) : m0u;
                m1 = p.mat.s1 ? __ldg(p.mat.p1 + (int64_t)e * p.mat.s1) : m1u;
            } else {
                m0 = p.mat.s0 ? xm0[el] : m0u;
                m1 = p.mat.s1 ? xm1[el] : m1u;
            }
            lame_elem<T>(p.mat, lsc, m0, m1, G.mu, G.lam);
            G.mu *= G.V;
            G.lam *= G.V;
        }
        T x[NV][D], H[D][D], P[D][D], psi = T(0);
        int bad = 0;
        if constexpr (OP == OP_TANGENT) {
            NhState<D, T> NS;
            if constexpr (MODEL == MODEL_NH) {
                T Hu[D][D];
                load_staged_field<D, T, T, 1>(ust + ust_sz, lv, 0, x);
                grad_of<D, T, T>(G, x, Hu);
                nh_state<D, T>(Hu, NS);
                bad = n_bad(NS.x);
            }
            load_staged_field<D, T, T, 1>(ust, lv, 0, x);
            grad_of<D, T, T>(G, x, H);
            dstress<D, MODEL, T, T>(G, NS, H, P);
        } else {
            load_staged_field<D, T, T, 1>(ust, lv, 0, x);
            grad_of<D, T, T>(G, x, H);
            stress<D, MODEL, T, T, HAS_PSI>(G, H, P, psi, bad);
        }
        if (MODEL == MODEL_NH && bad) {
            n_inv += bad;
            first_inv = min(first_inv, e);
        }
        if (HAS_PSI) {
            if (!isfinite(psi)) ++n_nonfin;
            wacc += psi;
            if (p.W_e) p.W_e[e] = psi;
        }
        if (HAS_FORCE) {
            T f[NV][D];
            forces<D, T, T>(G, P, f);
#pragma unroll
            for (int a = 0; a < NV; ++a)
#pragma unroll
                for (int i = 0; i < D; ++i) fb[(a * D + i) * EB + el] = f[a][i];
            if (!HAS_PSI && !isfinite(f[0][0])) ++n_nonfin;
        }
    }
    double dot_acc = 0.0, fsum = 0.0;
    if (HAS_FORCE || p.f_ext) {
        __syncthreads();
        // ---------------- phase 2: block-local CSR gather, thread per occurrence
        for (int oi = tid; oi < no; oi += NT) {
            const int word = socc[oi];
            const int node = word & OCC_NODE_MASK;
            if (HAS_FORCE) {
                T acc[D];
#pragma unroll
                for (int i = 0; i < D; ++i) acc[i] = T(0);
                const int k1 = soe[oi + 1];
                for (int k = soe[oi]; k < k1; ++k) {
                    const int slot = sle[k];   // a EB + el
                    const int a = (slot >= EB) + (slot >= 2 * EB) + (D == 3 ? (slot >= 3 * EB) : 0);
                    PFEM_DCHECK(slot < NV * EB && slot - a * EB < ne);
                    const T* q = fb + slot + a * (D - 1) * EB;   // row a d, column el
#pragma unroll
                    for (int i = 0; i < D; ++i) acc[i] += q[i * EB];
                }
                if (word & (OCC_NONOWNER | OCC_EARLIER)) {
                    const int slot = sseg[oi];
                    PFEM_DCHECK(slot >= 0 && slot < p.n_seg_total);
                    T* dst = p.partial + (int64_t)slot * D;
#pragma unroll
                    for (int i = 0; i < D; ++i) dst[i] = acc[i];
                } else {
                    const int64_t nb = (int64_t)node * D;
#pragma unroll
                    for (int i = 0; i < D; ++i) {
                        T val = acc[i];
                        if (OP == OP_TANGENT && MASKED && __ldg(p.mask + nb + i)) val = __ldg(p.v + nb + i);
                        p.out[nb + i] = out_value(p, nb + i, val);
                        if (cgdot) dot_acc += (double)__ldg(p.v + nb + i) * (double)val;
                    }
                }
            }
            if (HAS_PSI && p.f_ext && !(word & OCC_NONOWNER)) {
                const int64_t nb = (int64_t)node * D;
                double w = 0.0;
#pragma unroll
                for (int i = 0; i < D; ++i) w += (double)__ldg(p.f_ext + nb + i) * (double)__ldg(p.u + nb + i);
                fsum += w;
            }
        }
    }
    // ---------------- per-block sums (fixed order: warp shuffle tree, warps ascending)
    if (HAS_PSI || cgdot) {
        if (HAS_PSI) {
            const double a = (double)warp_sum_t<T>(wacc);
            const double f2 = p.f_ext ? warp_sum(fsum) : 0.0;
            if (lane == 0) { s_red[warp][0] = a; s_red[warp][1] = f2; }
        }
        if (cgdot) {
            const double d2 = warp_sum(dot_acc);
            if (lane == 0) s_red[warp][2] = d2;
        }
        __syncthreads();
        if (warp == 0) {
            if (HAS_PSI && lane < 2) {
                double r = 0.0;
                for (int w = 0; w < NT / 32; ++w) r += s_red[w][lane];
                p.blk_sum[(int64_t)lane * p.n_blocks + b] = r;
            }
            if (cgdot && lane == 31) {
                double r = 0.0;
                for (int w = 0; w < NT / 32; ++w) r += s_red[w][2];
                p.blk_sum[(int64_t)2 * p.n_blocks + b] = r;
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

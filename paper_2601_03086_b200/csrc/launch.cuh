// launch.cuh — host-side dispatch of the element kernels (template selection, smem
// sizing, grid), instantiated per (dim, dtype) in asm_{2,3}{f,d}.cu.
#pragma once

#include <algorithm>
#include <cstdlib>

#include "assemble.cuh"
#include "assemble_direct.cuh"
#include "assemble_dt.cuh"

#ifndef PFEM_DT
#define PFEM_DT 1   // fp64 single-sample calls: the in-place form (assemble_dt.cuh; config 4 K.v 131.3 -> 115.6 us);
                    // 0 = k_assemble_direct (A/B builds)
#endif

namespace pfem {
template <class T>
inline int P_nfix(const AsmParams<T>& p) { return p.n_fix; }
}  // namespace pfem

namespace pfem {

struct Call {
    const pfem_mesh* m;
    const Plan* P;
    int op, model, mode, S;
    int64_t sstride;
    pfem_material mat;
    const void* u;
    const void* v;
    const uint8_t* mask;
    const void* f_ext;
    void* W_e;
    void* totals;
    void* out;
    pfem_flags* flags;
    void* ws;
    size_t ws_bytes;
    cudaStream_t stream;
    CgState* cg;
    const void* cg_r;      // pipelined CG direction update (AsmParams::cg_r)
    const void* cg_pold;
    const void* cg_dinv;
    // pretraining-loss epilogue (pretrain.cu): out = phi (.) (f_int - f_ext) / (S K), loss
    int ep;
    const void* ep_phi;
    double* ep_loss;
};

template <class T>
AsmParams<T> make_params(const Call& c) {
    const Plan& P = *c.P;
    AsmParams<T> p;
    p.E = P.n_elems;
    p.N = P.n_nodes;
    p.S = c.S;
    p.K = P.n_parts;
    p.sstride = c.sstride;
    p.conn = c.m->conn;
    p.grad = (const T*)c.m->grad;
    p.vol = (const T*)c.m->vol;
    p.coords = c.m->coords;
    p.otf = (c.m->geometry == PFEM_GEOMETRY_ON_THE_FLY && c.mode == PFEM_ASSEMBLE_CSR) ? 1 : 0;
    p.mat.kind = c.mat.kind;
    p.mat.p0 = (const T*)c.mat.p0;
    p.mat.p1 = (const T*)c.mat.p1;
    p.mat.s0 = c.mat.stride0;
    p.mat.s1 = c.mat.stride1;
    p.u = (const T*)c.u;
    p.v = (const T*)c.v;
    p.mask = c.mask;
    p.f_ext = (const T*)c.f_ext;
    p.W_e = (T*)c.W_e;
    p.totals = (T*)c.totals;
    p.out = (T*)c.out;
    p.uflags = c.flags;
    p.n_blocks = P.n_blocks;
    p.n_occ = P.n_occ;
    p.eb_max = P.eb_max;
    p.n_chunks = P.n_chunks;
    p.blk_elem = P.blk_elem;
    p.blk_chunk = P.blk_chunk;
    p.chunk_blk = P.chunk_blk;
    p.part_chunk = P.part_chunk;
    p.blk_occ = P.blk_occ;
    p.blk_min_dep = P.blk_min_dep;
    p.part_blk = P.part_blk;
    p.occ_node = P.occ_node;
    p.occ_ent_ptr = P.occ_ent_ptr;
    p.loc_ent = P.loc_ent;
    p.node_occ_ptr = P.node_occ_ptr;
    p.node_occ = P.node_occ;
    p.blk_fix = P.blk_fix;
    p.fix_occ = P.fix_occ;
    p.fix_node = P.fix_node;
    p.fix_src_ptr = P.fix_src_ptr;
    p.fix_src = P.fix_src;
    p.occ_seg = P.occ_seg;
    p.n_fix = P.n_fix;
    p.n_seg_total = P.n_seg;
    p.perm = P.elem_perm != nullptr;
    p.rec = P.rec;
    p.rec_base = 0;
    p.rec_end = P.rec.bytes;
    p.recs = P.recs;
    const WsLayout L = ws_layout(P, c.S, sizeof(T));
    char* w = (char*)c.ws;
    p.ctr = (Counters*)(w + L.counters);
    p.blk_sum = (double*)(w + L.blk_sum);
    p.chunk_sum = (double*)(w + L.chunk_sum);
    p.partial = (T*)(w + L.partial);
    p.part_cnt = (int32_t*)(w + L.part_cnt);
    p.cg = c.cg;
    p.cg_r = (const T*)c.cg_r;
    p.cg_pold = (const T*)c.cg_pold;
    p.cg_dinv = (const T*)c.cg_dinv;
    p.ep = c.ep;
    p.ep_phi = (const T*)c.ep_phi;
    p.ep_scale = (T)(1.0 / ((double)c.S * (double)P.n_parts));
    p.ep_loss = c.ep_loss;
    p.lag = 0;
    return p;
}

constexpr int NTB_FINISH = 256;   // kernel B threads per CTA (128 / 512 measured no better)
template <class T>
constexpr int direct_nt() { return sizeof(T) == 4 ? 128 : 256; }   // direct kernel threads per CTA (measured)

template <int D, int MODEL, class T, int OP, int ST, bool MASKED, int NT, bool PERM, bool OTF>
pfem_status launch_direct(AsmParams<T> p, cudaStream_t s) {
    constexpr bool HAS_FORCE = OP != OP_ENERGY;
    constexpr int NFd = (OP == OP_TANGENT && MODEL == MODEL_NH) ? 2 : 1;
    const size_t smem0 = ((NFd * (size_t)p.rec.ocap * D * ST * sizeof(T) + (sizeof(T) == 4 ? 0 : 2 * (size_t)(D + 1) * p.rec.eb) +
                           15) & ~size_t(15)) +
                         (HAS_FORCE ? (size_t)ST * D * (D + 1) * p.rec.eb * sizeof(T) : 0);
    // on-the-fly geometry: the block's vertex coordinates [ocap][D] fp64 after everything else
    const size_t smem = OTF ? ((smem0 + 15) & ~size_t(15)) + (size_t)p.rec.ocap * D * sizeof(double) : smem0;
    auto kd = k_assemble_direct<D, MODEL, T, OP, ST, MASKED, NT, PERM, OTF>;
    static size_t configured = 0;
    static int pf_auto = 0;
    if (smem > configured || pf_auto == 0) {
        PFEM_CUDA_TRY(cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1)));
        configured = std::max(configured, smem);
        int dev = 0, nsm = 0, per_sm = 0;
        PFEM_CUDA_TRY(cudaGetDevice(&dev));
        PFEM_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        PFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kd, NT, smem));
        pf_auto = std::max(1, std::min(per_sm, 2) * nsm);   // measured: a deeper prefetch evicts
    }
    p.lag = pf_auto;   // L2 prefetch distance in blocks (~ one wave ahead)
    kd<<<std::max(1, p.n_blocks), NT, smem, s>>>(p);
    PFEM_LAUNCH_CHECK("k_assemble_direct");
    return PFEM_OK;
}

// the in-place single-sample form (assemble_dt.cuh).  Returns 1 when launched, 0 when the plan's
// record layout or the shared-memory size does not suit it (the caller then takes
// k_assemble_direct), or a negative pfem_status
template <int D, int MODEL, class T, int OP, bool MASKED, int NT, bool PERM>
int launch_dt(AsmParams<T> p, cudaStream_t s) {
    constexpr int NFd = (OP == OP_TANGENT && MODEL == MODEL_NH) ? 2 : 1;
    const DtLayout L = dt_layout(p.rec, D, (int)sizeof(T), NFd);
    if (!L.ok) return 0;
    auto kd = k_assemble_dt<D, MODEL, T, OP, MASKED, NT, PERM>;
    static size_t configured = 0;
    static int pf_auto = 0;
    const size_t smem = L.total;
    if (smem > configured || pf_auto == 0) {
        int dev = 0, nsm = 0, per_sm = 0, maxsm = 0;
        PFEM_CUDA_TRY(cudaGetDevice(&dev));
        PFEM_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        PFEM_CUDA_TRY(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        if (smem > (size_t)maxsm) return 0;
        PFEM_CUDA_TRY(cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = std::max(configured, smem);
        PFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kd, NT, smem));
        if (per_sm < 1) return 0;
        pf_auto = std::max(1, std::min(per_sm, 2) * nsm);   // L2 prefetch distance (~ one wave)
    }
    p.lag = pf_auto;
    kd<<<std::max(1, p.n_blocks), NT, smem, s>>>(p);
    PFEM_LAUNCH_CHECK("k_assemble_dt");
    return 1;
}

template <int D, int MODEL, class T, int OP, int ST, bool MASKED>
pfem_status launch_csr(AsmParams<T> p, cudaStream_t s) {
    constexpr bool HAS_FORCE = OP != OP_ENERGY;
    constexpr bool HAS_PSI = OP == OP_ENERGY || OP == OP_ENERGY_RESIDUAL;
    constexpr int EB = EbOf<D>::value;
    constexpr int NT = STAGED_NT;
    constexpr int NF = (OP == OP_TANGENT && MODEL == MODEL_NH) ? 2 : 1;   // staged fields (single buffer)
    // kernel A form: direct (one CTA per block, small shared memory) for single-sample calls,
    // where the kernel is bound by memory latency and occupancy pays; staged persistent
    // otherwise (several samples per element: arithmetic-heavy, staging amortised).
    // Blocks larger than the staged kernel's compile-time capacity always take the direct form.
    // (the staged form reads the record with its compile-time stride EB)
    // (CG products, p.cg set, always take the direct form: the staged kernel has no fused p.q)
    // (on-the-fly geometry is a direct-form option)
    const bool direct = p.otf || p.eb_max > EB || p.rec.eb != EB || p.cg != nullptr || p.S == 1;
    if (direct) {
        pfem_status st = PFEM_OK;
        int done = 0;
        if (PFEM_DT && ST == 1 && sizeof(T) == 8 && !p.otf) {   // (fp32 config 5: 70.5 -> 74.1 us, not taken)
            done = p.perm ? launch_dt<D, MODEL, T, OP, MASKED, direct_nt<T>(), true>(p, s)
                          : launch_dt<D, MODEL, T, OP, MASKED, direct_nt<T>(), false>(p, s);
            if (done < 0) return (pfem_status)done;
        }
        if (done) {
        } else if (p.otf)
            st = p.perm ? launch_direct<D, MODEL, T, OP, ST, MASKED, direct_nt<T>(), true, true>(p, s)
                        : launch_direct<D, MODEL, T, OP, ST, MASKED, direct_nt<T>(), false, true>(p, s);
        else
            st = p.perm ? launch_direct<D, MODEL, T, OP, ST, MASKED, direct_nt<T>(), true, false>(p, s)
                        : launch_direct<D, MODEL, T, OP, ST, MASKED, direct_nt<T>(), false, false>(p, s);
        if (st != PFEM_OK) return st;
    } else {
        // the staged copy (RecLayout order) skips conn and ent_pos: every work item stages its
        // fields (and the NH state u); the element-major force buffer is gathered through loc_ent
        p.rec_base = p.rec.g;
        p.rec_end = p.rec.bytes;
        const size_t smem = 2 * (size_t)(p.rec_end - p.rec_base) +
                            (((p.mat.s0 | p.mat.s1) != 0) ? 4 * EB * sizeof(T) : 0) +
                            (size_t)NF * p.rec.ocap * D * ST * sizeof(T) +
                            (HAS_FORCE ? (size_t)ST * D * (D + 1) * EB * sizeof(T) : 0);
        const int fx = (HAS_PSI && p.f_ext) ? 1 : 0;
        auto kern = fx ? k_assemble<D, MODEL, T, OP, ST, MASKED, EB, NT, HAS_PSI> : k_assemble<D, MODEL, T, OP, ST, MASKED, EB, NT, false>;
        static int resident_[2] = {0, 0};   // per instantiation: co-resident CTAs (persistent grid)
        static size_t configured_[2] = {0, 0};
        int& resident = resident_[fx];
        size_t& configured = configured_[fx];
        if (resident == 0 || smem > configured) {
            PFEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            configured = smem;
            int dev = 0, nsm = 0, per_sm = 0;
            PFEM_CUDA_TRY(cudaGetDevice(&dev));
            PFEM_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
            PFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
            if (per_sm < 1) {
                set_error("CSR kernel does not fit on an SM (block record too large)");
                return PFEM_ERR_CAPACITY;
            }
            resident = per_sm * nsm;
        }
        const int items = p.n_blocks * ((p.S + ST - 1) / ST);   // (block, sample chunk) work items
        const int grid = std::max(1, std::min(resident, items));
        kern<<<grid, NT, smem, s>>>(p);
        PFEM_LAUNCH_CHECK("k_assemble");
    }
    // kernel B: finish multi-block nodes + reductions (programmatic dependent launch)
    constexpr int NTB = NTB_FINISH;
    const int nsc = (p.S + ST - 1) / ST;
    const int n_items = HAS_FORCE ? P_nfix(p) * nsc : 0;
    int gridb = std::max({1, (n_items + NTB - 1) / NTB, 0});
    // few CTAs, grid-stride: every CTA ends with one atomic on the shared exit counter, and
    // thousands of same-address atomics serialise into a tail that idles the GPU
    static int cap_b = 0;
    if (cap_b == 0) {
        int dev = 0, nsm = 0;
        PFEM_CUDA_TRY(cudaGetDevice(&dev));
        PFEM_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        cap_b = 8 * nsm;   // (592 / 296 / 148 measured slower)
    }
    gridb = std::max(1, std::min(gridb, std::min(p.n_blocks, cap_b)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gridb);
    cfg.blockDim = dim3(NTB);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PFEM_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_node_finish<D, T, ST, MASKED, NTB>, p, HAS_PSI ? 1 : 0, n_items));
    count_launch();
    return PFEM_OK;
}

template <int D, int MODEL, class T, int OP, bool MASKED>
pfem_status dispatch_st(const AsmParams<T>& p, cudaStream_t s) {
    constexpr int STBIG = sizeof(T) == 4 ? 4 : 2;
    if (p.S > 1) return launch_csr<D, MODEL, T, OP, STBIG, MASKED>(p, s);
    return launch_csr<D, MODEL, T, OP, 1, MASKED>(p, s);
}

template <int D, int MODEL, class T, int OP, bool MASKED>
pfem_status run_colour(const Call& c, AsmParams<T> p) {
    constexpr bool HAS_FORCE = OP != OP_ENERGY;
    constexpr bool HAS_PSI = OP == OP_ENERGY || OP == OP_ENERGY_RESIDUAL;
    cudaStream_t s = c.stream;
    const Plan& P = *c.P;
    const WsLayout L = ws_layout(P, c.S, sizeof(T));
    T* wtmp = c.W_e ? (T*)c.W_e : (T*)((char*)c.ws + L.wtmp);
    if (HAS_FORCE) {
        const size_t row = sizeof(T) * (size_t)P.n_nodes * D;
        if (c.sstride == (int64_t)P.n_nodes * D) {
            PFEM_CUDA_TRY(cudaMemsetAsync(c.out, 0, row * c.S, s));
        } else {
            for (int q = 0; q < c.S; ++q)
                PFEM_CUDA_TRY(cudaMemsetAsync((char*)c.out + sizeof(T) * c.sstride * q, 0, row, s));
        }
    }
    const std::vector<int32_t>& cp = P.colour_ptr_host;
    for (size_t col = 0; col + 1 < cp.size(); ++col) {
        const int i0 = cp[col], i1 = cp[col + 1];
        if (i1 <= i0) continue;
        k_colour_pass<D, MODEL, T, OP, MASKED><<<(i1 - i0 + ASM_NT - 1) / ASM_NT, ASM_NT, 0, s>>>(
            p, c.m->colour_elems, i0, i1, wtmp);
        PFEM_LAUNCH_CHECK("k_colour_pass");
    }
    if (OP == OP_TANGENT && MASKED) {
        const int64_t n = (int64_t)P.n_nodes * D;
        k_mask_rows<D, T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c.S, P.n_nodes, c.sstride, c.mask, (const T*)c.v,
                                                                        (T*)c.out);
        PFEM_LAUNCH_CHECK("k_mask_rows");
    }
    const int want = HAS_PSI && c.totals ? 1 : 0;
    k_colour_totals<D, T><<<want ? c.S * P.n_parts : 1, ASM_NT, 0, s>>>(p, P.part_elem, P.part_node, wtmp, want);
    PFEM_LAUNCH_CHECK("k_colour_totals");
    return PFEM_OK;
}

template <int D, int MODEL, class T, int OP, bool MASKED>
pfem_status run_op(const Call& c) {
    AsmParams<T> p = make_params<T>(c);
    if (c.mode == PFEM_ASSEMBLE_COLOUR && OP != OP_ENERGY) return run_colour<D, MODEL, T, OP, MASKED>(c, p);
    if (c.mode == PFEM_ASSEMBLE_COLOUR) return run_colour<D, MODEL, T, OP, MASKED>(c, p);
    return dispatch_st<D, MODEL, T, OP, MASKED>(p, c.stream);
}

template <int D, int MODEL, class T>
pfem_status run_model(const Call& c) {
    switch (c.op) {
        case OP_ENERGY: return run_op<D, MODEL, T, OP_ENERGY, false>(c);
        case OP_ENERGY_RESIDUAL: return run_op<D, MODEL, T, OP_ENERGY_RESIDUAL, false>(c);
        case OP_RESIDUAL: return run_op<D, MODEL, T, OP_RESIDUAL, false>(c);
        case OP_TANGENT:
            return c.mask ? run_op<D, MODEL, T, OP_TANGENT, true>(c) : run_op<D, MODEL, T, OP_TANGENT, false>(c);
    }
    set_error("bad op");
    return PFEM_ERR_ARG;
}

template <class T>
pfem_status run_quad(const Call& c);   // quad.cu: Q4 / Q8 elements (§8(f) row f4)

template <int D, class T>
pfem_status run_assemble(const Call& c) {
    if (c.P->elem_type != PFEM_ELEM_SIMPLEX) return run_quad<T>(c);
    return c.model == MODEL_NH ? run_model<D, MODEL_NH, T>(c) : run_model<D, MODEL_LINEAR, T>(c);
}

// explicit instantiations live in asm_*.cu
extern template pfem_status run_assemble<2, float>(const Call&);
extern template pfem_status run_assemble<2, double>(const Call&);
extern template pfem_status run_assemble<3, float>(const Call&);
extern template pfem_status run_assemble<3, double>(const Call&);

}  // namespace pfem

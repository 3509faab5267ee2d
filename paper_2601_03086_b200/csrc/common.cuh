// common.cuh — shared host/device plumbing of libpfem (errors, plan layout, workspace
// layout, memory-model helpers).  Product code; no oracle code is included anywhere.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <algorithm>
#include <vector>

#include "../../include/pfem.h"

namespace pfem {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg, int64_t index = -1);
pfem_status cuda_status(cudaError_t e, const char* what);
void count_launch(int n = 1);

#define PFEM_CUDA_TRY(expr)                                             \
    do {                                                                \
        cudaError_t _e = (expr);                                        \
        if (_e != cudaSuccess) return ::pfem::cuda_status(_e, #expr);   \
    } while (0)

#define PFEM_LAUNCH_CHECK(name)                                         \
    do {                                                                \
        ::pfem::count_launch();                                         \
        cudaError_t _e = cudaGetLastError();                            \
        if (_e != cudaSuccess) return ::pfem::cuda_status(_e, name);    \
    } while (0)

// ------------------------------------------------------------------ plan
// Occurrence kind bits packed in occ_node (node ids < 2^30).
constexpr int32_t OCC_NODE_MASK = 0x1fffffff;  // prepare rejects n_nodes >= 2^29
constexpr int32_t OCC_NONOWNER = 0x40000000;   // another (later) block owns the node
constexpr int32_t OCC_EARLIER = 0x20000000;    // owner, and earlier blocks hold partials

// ------------------------------------------------------------------ packed block records
// The plan keeps, per element block, one contiguous 16-byte-aligned record holding
// everything phase 1 and phase 2 read from HBM about the block, so a single TMA bulk copy
// (cp.async.bulk) stages it into shared memory:
//   conn [EB][d+1] int32 | ent_pos [EB][d+1] uint16 (inverse of loc_ent: the block-CSR entry
//   of each element vertex) | grad [d*d][EB] T | vol [EB] T | eid [EB] int32 (input element
//   id of each position: the plan may order elements for locality) | occ_node [OCAP] int32 |
//   occ_ent [OCAP+1] uint16 (block-relative entry offsets) | lconn [EB][d+1] uint16
//   (block-local occurrence index of each element vertex) | occ_seg [OCAP] int32 (node-major
//   segment slot of a multi-block node's occurrence, -1 if the node is finished inside the
//   block) | occ_perm [OCAP] uint16 (the block's occurrences ordered by descending entry count,
//   ties by index: the staged kernel's phase-2 thread order, so each warp gathers occurrences
//   of similar length) | loc_ent [(d+1) EB] uint16 (each block-CSR entry's force-buffer slot
//   a * EB + el)
// The order lets every kernel form read one contiguous range: fp32 forms (force buffer in
// entry order) [ent_pos, loc_ent), fp64 forms (loc_ent gather) [g, end), and the gathering
// staged forms start at conn.
struct RecLayout {
    int eb = 0, ocap = 0;
    uint32_t conn = 0, g = 0, vol = 0, eid = 0, occ_node = 0, occ_ent = 0, loc_ent = 0, lconn = 0, occ_seg = 0, ent_pos = 0,
             occ_perm = 0, bytes = 0;
};

inline RecLayout rec_layout(int D, size_t tsize, int eb, int ocap, bool with_eid) {
    RecLayout L;
    L.eb = eb;
    L.ocap = ocap;
    size_t o = 0;
    auto take = [&](size_t b) { size_t at = o; o += (b + 15) / 16 * 16; return (uint32_t)at; };
    L.conn = take(4 * (size_t)(D + 1) * eb);
    L.ent_pos = take(2 * (size_t)(D + 1) * eb);
    L.g = take(tsize * D * D * (size_t)eb);
    L.vol = take(tsize * (size_t)eb);
    L.eid = take(with_eid ? 4 * (size_t)eb : 0);   // identity order: no ids stored
    L.occ_node = take(4 * (size_t)ocap);
    L.occ_ent = take(2 * (size_t)(ocap + 1));
    L.lconn = take(2 * (size_t)(D + 1) * eb);
    L.occ_seg = take(4 * (size_t)ocap);
    L.occ_perm = take(2 * (size_t)ocap);   // occurrences by descending entry count (phase-2 balance)
    L.loc_ent = take(2 * (size_t)(D + 1) * eb);
    L.bytes = (uint32_t)o;
    return L;
}

struct Plan {
    uint64_t serial = 0;              // unique per prepared plan in this process (workspace caches key on it)
    int32_t dim = 0, n_nodes = 0, n_elems = 0, n_parts = 0;
    int32_t elem_type = 0;            // pfem_elem_type; quadrilaterals have no block plan (quad.cu)
    int32_t nv = 0;                   // nodes per element
    void* quad_geo = nullptr;         // [E][nq][2 nv + 1] dN/dX and w det J per Gauss point (dtype)
    int32_t* quad_pos = nullptr;      // [E * nv] CSR entry of every (element, node)
    void* pool_quad = nullptr;
    int32_t n_blocks = 0, n_occ = 0, eb_max = 0;
    int32_t* blk_elem = nullptr;      // [n_blocks+1] in plan positions (see elem_perm)
    int32_t elem_order = 0;           // 0 input order, 1 locality (Morton) order of the positions
    int32_t* elem_perm = nullptr;     // [n_elems] position -> input element id (null: identity)
    int32_t* conn_p = nullptr;        // [n_elems][d+1] connectivity in position order (null: conn)
    int32_t* csr_ptr_p = nullptr;     // node -> (position, slot) CSR (null: the mesh's CSR)
    int32_t* csr_ent_p = nullptr;
    void* pool_perm = nullptr;
    int32_t* blk_occ = nullptr;       // [n_blocks+1]
    int32_t* blk_min_dep = nullptr;   // [n_blocks] lowest block holding a partial this block
                                      // needs (== b if none); the block waits for [min_dep, b)
    int32_t* part_blk = nullptr;      // [n_parts+1]
    int32_t n_chunks = 0;             // reduction chunks (<= CHUNK consecutive blocks, inside a part)
    int32_t* blk_chunk = nullptr;     // [n_blocks]
    int32_t* chunk_blk = nullptr;     // [n_chunks+1]
    int32_t* part_chunk = nullptr;    // [n_parts+1]
    std::vector<int32_t> colour_ptr_host;  // [n_colours+1] (colour-mode launches)
    int32_t* part_node = nullptr;     // [n_parts+1] (device copy, always present)
    int32_t* part_elem = nullptr;     // [n_parts+1] (device copy, always present)
    int32_t* occ_node = nullptr;      // [n_occ] node | kind bits
    int32_t* occ_ent_ptr = nullptr;   // [n_occ+1] offsets into loc_ent
    uint16_t* loc_ent = nullptr;      // [(dim+1)*n_elems] local entry ids, grouped by occurrence
    int32_t* node_occ_ptr = nullptr;  // [n_nodes+1]
    int32_t* node_occ = nullptr;      // [n_occ] occurrence ids sorted by (node, block)
    int32_t n_fix = 0;                // owned nodes with partials in earlier blocks
    int32_t* blk_fix = nullptr;       // [n_blocks+1] offsets into fix_occ
    int32_t* fix_occ = nullptr;       // [n_fix] occurrence ids (fix-up list of each block)
    int32_t* fix_node = nullptr;      // [n_fix] node id of each fix entry
    int32_t* fix_src_ptr = nullptr;   // [n_fix+1] offsets into fix_src
    int32_t* fix_src = nullptr;       // all occurrences of the node, ascending block (own last)
    int32_t* occ_seg = nullptr;       // [n_occ] node-major segment slot (fix_src position), -1 single
    int32_t n_seg = 0;                // segments of multi-block nodes (= fix_src_ptr[n_fix])
    void* pool_fix = nullptr;
    void* pool_src = nullptr;
    RecLayout rec;                    // packed block records (one bulk copy per block)
    unsigned char* recs = nullptr;    // [n_blocks][rec.bytes]
    void* pool_rec = nullptr;
    void* pool = nullptr;             // single allocation backing all of the above
};

// ------------------------------------------------------------------ workspace layout
// [ Counters | part_cnt[n_parts] | blk_sum[2S+2][n_blocks] (double) | chunk_sum[2S+1][n_chunks] (double) |
//   partial[n_seg][S][d] (T) | colour-mode W [S][E] (T) ]
// The zero-at-rest counters (Counters, part_cnt) sit at offsets that depend only on the plan, so
// one workspace sized for the largest sample count may serve calls with any S.
struct Counters {
    int32_t ticket;
    int32_t done;
    int32_t epoch;
    int32_t n_inv;
    int32_t first_inv;     // stored as INT32_MAX - first (atomicMax; 0 = none) so zero-fill is valid
    int32_t n_nonfinite;
    int32_t exit_count;
    int32_t fix_ticket;
    int32_t pad[8];
};

struct WsLayout {
    size_t counters, part_cnt, blk_sum, chunk_sum, partial, wtmp, total;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

inline WsLayout ws_layout(const Plan& p, int S, size_t tsize) {
    WsLayout L;
    size_t o = 0;
    L.counters = o; o += align_up(sizeof(Counters), 256);
    L.part_cnt = o; o += align_up(sizeof(int32_t) * (size_t)(p.n_parts + 1), 256);   // reduced chunks per part
    L.blk_sum = o;  o += align_up(sizeof(double) * (2 * (size_t)S + 2) * (p.n_blocks + 1), 256);
    L.chunk_sum = o;  o += align_up(sizeof(double) * (2 * (size_t)S + 1) * (p.n_chunks + 1), 256);
    // segments of multi-block nodes (simplices) / nodal forces at their CSR entries (quadrilaterals)
    const size_t seg = tsize * (size_t)S * std::max(p.n_seg, 1) * p.dim;
    const size_t qeb = p.elem_type ? tsize * (size_t)S * p.n_elems * p.nv * 2 : 0;
    L.partial = o;  o += align_up(std::max(seg, qeb), 256);
    L.wtmp = o;     o += align_up(tsize * (size_t)S * p.n_elems, 256);
    L.total = o;
    return L;
}

// ------------------------------------------------------------------ checked builds
// PFEM_CHECKED (tools/checked_tests.sh): every plan-derived index is bounds-checked on the device
// and a violation traps (the kernel faults, the call returns PFEM_ERR_CUDA) — the stand-in for
// compute-sanitizer, which this pool does not offer.  Release builds compile the checks out.
#ifdef PFEM_CHECKED
#define PFEM_DCHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define PFEM_DCHECK(cond) do { } while (0)
#endif

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ float ld_relaxed(const float* p) {
    float v;
    asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ld_relaxed(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed_i(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace pfem

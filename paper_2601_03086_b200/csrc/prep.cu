// prep.cu — one-time mesh preparation on the GPU (§8 row a1):
//   K1 geometry (J_e^{-1} rows = grad N_a, V_e = |det J_e|/d!; App. B)
//   K2 node -> (element, slot) CSR (count / scan / fill / per-row sort -> ascending (e, a))
//   K3 greedy first-fit colouring in element order (ticketed warps, dependency-driven)
//      + colour-sorted element list (stable radix sort on the colour key)
//   plan: element blocks, block-local CSR (smem bitonic sort of (node, entry) keys),
//      node occurrences with ownership / earlier-partial kinds, node-major occurrence list.
#include <atomic>
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "element.cuh"

namespace pfem {

// ------------------------------------------------------------------ validation
__global__ void k_check_conn(int nv, int E, int N, const int32_t* __restrict__ conn, int* bad) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (int64_t)E * nv) return;
    int v = conn[k];
    if (v < 0 || v >= N) atomicMin(bad, (int)(k / nv));
}

// ------------------------------------------------------------------ K1 geometry
template <int D, class T>
__global__ void k_geometry(int E, const double* __restrict__ X, const int32_t* __restrict__ conn,
                           T* __restrict__ grad, T* __restrict__ vol, int* n_negative,
                           int* first_degenerate) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    int v[D + 1];
#pragma unroll
    for (int a = 0; a <= D; ++a) v[a] = conn[(int64_t)e * (D + 1) + a];
    double Xv[D + 1][D];
#pragma unroll
    for (int a = 0; a <= D; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) Xv[a][i] = X[(int64_t)v[a] * D + i];
    double eprod = 1.0;
#pragma unroll
    for (int a = 1; a <= D; ++a) {
        double l2 = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const double dx = Xv[a][i] - Xv[0][i];
            l2 += dx * dx;
        }
        eprod *= sqrt(l2);
    }
    double inv[D][D];
    const double det = geometry_of<D>(Xv, inv);
    if (!(fabs(det) > 64.0 * 2.220446049250313e-16 * eprod)) {
        atomicMin(first_degenerate, e);
        return;
    }
    if (det < 0) atomicAdd(n_negative, 1);
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int j = 0; j < D; ++j) grad[(int64_t)(a * D + j) * E + e] = (T)inv[a][j];
    vol[e] = (T)(fabs(det) / (D == 2 ? 2.0 : 6.0));
}

// ------------------------------------------------------------------ K2 CSR
__global__ void k_count(int64_t n, const int32_t* __restrict__ conn, int32_t* cnt) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) atomicAdd(&cnt[conn[k]], 1);
}

__global__ void k_csr_fill(int64_t n, const int32_t* __restrict__ conn, const int32_t* __restrict__ ptr,
                           int32_t* fill, int32_t* ent) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int v = conn[k];
    int pos = atomicAdd(&fill[v], 1);
    ent[ptr[v] + pos] = (int32_t)k;       // k = e*(d+1) + a
}

// per-row insertion sort -> ascending (e, a); rows hold at most a few dozen entries
__global__ void k_csr_sort_rows(int N, const int32_t* __restrict__ ptr, int32_t* ent) {
    int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    int b = ptr[n], e = ptr[n + 1];
    for (int i = b + 1; i < e; ++i) {
        int x = ent[i];
        int j = i - 1;
        while (j >= b && ent[j] > x) {
            ent[j + 1] = ent[j];
            --j;
        }
        ent[j + 1] = x;
    }
}

// ------------------------------------------------------------------ K3 colouring
// Greedy first-fit in ascending element id == Jones-Plassmann with priority -e.
// Warps take 32 consecutive elements by ticket; lane e resolves its lower neighbours
// (a prefix of each sorted CSR row) with a resumable cursor, waiting on lower ids that
// belong to earlier tickets (resident or finished) or lower lanes of the same warp, so
// the loop always progresses.  The colour value itself is the only payload (volatile).
__global__ void k_colour_greedy(int nv, int E, const int32_t* __restrict__ conn,
                                const int32_t* __restrict__ ptr, const int32_t* __restrict__ ent,
                                int32_t* colour, int* ticket, int max_colours, int* overflow) {
    const int lane = threadIdx.x & 31;
    volatile int32_t* vcol = colour;
    while (true) {
        int base = 0;
        if (lane == 0) base = atomicAdd(ticket, 32);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= E) return;
        const int e = base + lane;
        bool done = e >= E;
        unsigned long long used0 = 0ull, used1 = 0ull;
        int a = 0, k = -1;
        while (__any_sync(0xffffffffu, !done)) {
            bool blocked = false;
            if (!done) {
                while (a < nv) {
                    int n = conn[(int64_t)e * nv + a];
                    if (k < 0) k = ptr[n];
                    int kend = ptr[n + 1];
                    for (; k < kend; ++k) {
                        int f = ent[k] / nv;
                        if (f >= e) { k = kend; break; }
                        int c = vcol[f];
                        if (c < 0) { blocked = true; break; }
                        if (c < 64) used0 |= 1ull << c;
                        else used1 |= 1ull << (c - 64);
                    }
                    if (blocked) break;
                    ++a;
                    k = -1;
                }
                if (!blocked) {
                    // both masks full (all 128 colours taken below e): overflow, never a reused colour
                    int c = (~used0) ? __ffsll((long long)~used0) - 1 : ((~used1) ? 64 + __ffsll((long long)~used1) - 1 : 128);
                    if (c >= max_colours || c < 0) {
                        atomicMin(overflow, e);
                        c = max_colours - 1;       // keep going; prepare reports CAPACITY
                    }
                    vcol[e] = c;
                    done = true;
                }
            }
            __syncwarp();
            if (blocked) __nanosleep(64);
        }
    }
}

__global__ void k_colour_hist(int E, const int32_t* __restrict__ colour, int32_t* hist, int* maxc) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    int c = colour[e];
    atomicAdd(&hist[c], 1);
    atomicMax(maxc, c);
}

// exclusive scan of the (<= 129) colour counts; single thread, integer
__global__ void k_colour_ptr(int nc, const int32_t* __restrict__ hist, int32_t* cptr) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int s = 0;
    for (int c = 0; c < nc; ++c) {
        cptr[c] = s;
        s += hist[c];
    }
    cptr[nc] = s;
}

__global__ void k_iota(int n, int32_t* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

// ------------------------------------------------------------------ locality order
// order-preserving map of a double onto uint64 (for integer atomics min / max)
__device__ __forceinline__ unsigned long long dkey(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// bounding box of the nodes: bb[0..D) = min keys, bb[D..2D) = max keys
__global__ void k_bbox(int N, int D, const double* __restrict__ coords, unsigned long long* bb) {
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0ull, 0ull, 0ull};
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
        for (int j = 0; j < D; ++j) {
            const unsigned long long k = dkey(coords[(int64_t)n * D + j]);
            lo[j] = min(lo[j], k);
            hi[j] = max(hi[j], k);
        }
    for (int j = 0; j < D; ++j) {
        atomicMin(bb + j, lo[j]);
        atomicMax(bb + D + j, hi[j]);
    }
}

__device__ __forceinline__ uint32_t spread2(uint32_t x) {   // 15 bits -> every 2nd bit
    x &= 0x7fff;
    x = (x | (x << 8)) & 0x00ff00ffu;
    x = (x | (x << 4)) & 0x0f0f0f0fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}
__device__ __forceinline__ uint32_t spread3(uint32_t x) {   // 10 bits -> every 3rd bit
    x &= 0x3ff;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

// key = part << 32 | Morton code of the element centroid (30 bits, bounding box of the mesh)
__global__ void k_morton_keys(int E, int D, int K, const double* __restrict__ coords,
                              const int32_t* __restrict__ conn, const int32_t* __restrict__ part_elem,
                              const unsigned long long* __restrict__ bb, unsigned long long* key, int32_t* val) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int nv = D + 1;
    const int bits = D == 3 ? 10 : 15;
    uint32_t code = 0;
    for (int j = 0; j < D; ++j) {
        double c = 0.0;
        for (int a = 0; a < nv; ++a) c += coords[(int64_t)conn[(int64_t)e * nv + a] * D + j];
        c /= nv;
        const double lo = dkey_inv(bb[j]), hi = dkey_inv(bb[D + j]);
        const double t = hi > lo ? (c - lo) / (hi - lo) : 0.0;
        const uint32_t q = (uint32_t)min((double)((1 << bits) - 1), max(0.0, t * (double)(1 << bits)));
        code |= (D == 3 ? spread3(q) : spread2(q)) << j;
    }
    int part = 0;
    if (K > 1) {
        int lo = 0, hi = K - 1;   // last k with part_elem[k] <= e
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (part_elem[mid] <= e) lo = mid;
            else hi = mid - 1;
        }
        part = lo;
    }
    key[e] = ((unsigned long long)part << 32) | code;
    val[e] = e;
}

__global__ void k_gather_conn(int E, int nv, const int32_t* __restrict__ perm, const int32_t* __restrict__ conn,
                              int32_t* conn_p) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (int64_t)E * nv) return;
    const int64_t i = k / nv, a = k - i * nv;
    conn_p[k] = conn[(int64_t)perm[i] * nv + a];
}

// ------------------------------------------------------------------ plan
__device__ __forceinline__ int block_of(int e, const int32_t* __restrict__ blk_elem, int nb) {
    int lo = 0, hi = nb;     // blk_elem[lo] <= e < blk_elem[hi]
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (blk_elem[mid] <= e) lo = mid;
        else hi = mid;
    }
    return lo;
}

// number of distinct blocks touching each node (its CSR row is sorted by element)
__global__ void k_node_occ_count(int N, int nv, const int32_t* __restrict__ ptr,
                                 const int32_t* __restrict__ ent, const int32_t* __restrict__ blk_elem,
                                 int nb, int32_t* cnt) {
    int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    int c = 0, last = -1;
    for (int k = ptr[n]; k < ptr[n + 1]; ++k) {
        int b = block_of(ent[k] / nv, blk_elem, nb);
        if (b != last) { ++c; last = b; }
    }
    cnt[n] = c;
}

constexpr int PLAN_THREADS = 512;
constexpr int PLAN_MAX_KEYS = 4096;
constexpr int CHUNK_BLOCKS = 32;   // == CHUNK of assemble.cuh

// Per block: bitonic-sort the (node << 16 | local entry) keys of its elements in shared
// memory; runs of equal node = occurrences, in ascending node order; inside a run the
// local entries ascend = CSR order restricted to the block.
// mode 0: count occurrences -> occ_cnt[b], fix-ups -> fix_cnt[b], min_dep[b]
// mode 1: fill occ_node, occ_ent_ptr, loc_ent, node_occ, fix_occ (the block's owned nodes
//         with partials in earlier blocks, ascending node order)
__global__ void __launch_bounds__(PLAN_THREADS)
k_block_build(int mode, int nv, int nb, const int32_t* __restrict__ blk_elem,
              const int32_t* __restrict__ conn, const int32_t* __restrict__ csr_ptr,
              const int32_t* __restrict__ csr_ent, int32_t* occ_cnt, int32_t* fix_cnt, int32_t* min_dep,
              const int32_t* __restrict__ blk_occ, int32_t* occ_node, int32_t* occ_ent_ptr,
              uint16_t* loc_ent, const int32_t* __restrict__ node_occ_ptr, int32_t* node_occ,
              const int32_t* __restrict__ blk_fix, int32_t* fix_occ) {
    __shared__ unsigned long long key[PLAN_MAX_KEYS];
    __shared__ uint16_t runid[PLAN_MAX_KEYS];
    __shared__ uint8_t sfix[PLAN_MAX_KEYS];
    __shared__ int32_t s_scan[PLAN_THREADS];
    __shared__ int32_t s_mindep;
    const int b = blockIdx.x;
    const int e0 = blk_elem[b], e1 = blk_elem[b + 1];
    const int cnt = (e1 - e0) * nv;
    int P = 1;
    while (P < cnt) P <<= 1;
    for (int i = threadIdx.x; i < P; i += PLAN_THREADS) {
        if (i < cnt) {
            int node = conn[(int64_t)e0 * nv + i];
            key[i] = ((unsigned long long)(unsigned)node << 16) | (unsigned)i;
        } else {
            key[i] = ~0ull;
        }
    }
    if (threadIdx.x == 0) s_mindep = b;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += PLAN_THREADS) {
                int ixj = i ^ j;
                if (ixj > i) {
                    unsigned long long x = key[i], y = key[ixj];
                    bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        key[i] = y;
                        key[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
    // run starts and their ranks (block-wide scan over per-thread chunk counts)
    const int per = (cnt + PLAN_THREADS - 1) / PLAN_THREADS;
    const int lo = threadIdx.x * per, hi = min(cnt, lo + per);
    int local = 0;
    for (int i = lo; i < hi; ++i)
        local += (i == 0 || (key[i] >> 16) != (key[i - 1] >> 16)) ? 1 : 0;
    s_scan[threadIdx.x] = local;
    __syncthreads();
    for (int off = 1; off < PLAN_THREADS; off <<= 1) {
        int v = threadIdx.x >= off ? s_scan[threadIdx.x - off] : 0;
        __syncthreads();
        s_scan[threadIdx.x] += v;
        __syncthreads();
    }
    int r = s_scan[threadIdx.x] - local;     // exclusive
    for (int i = lo; i < hi; ++i) {
        if (i == 0 || (key[i] >> 16) != (key[i - 1] >> 16)) ++r;
        runid[i] = (uint16_t)(r - 1);
    }
    const int n_occ_b = s_scan[PLAN_THREADS - 1];
    __syncthreads();
    // per occurrence: kind, earlier-block rank, min dep
    for (int i = threadIdx.x; i < cnt; i += PLAN_THREADS) {
        bool start = (i == 0 || (key[i] >> 16) != (key[i - 1] >> 16));
        int node = (int)(key[i] >> 16);
        if (mode == 1) loc_ent[(int64_t)e0 * nv + i] = (uint16_t)(key[i] & 0xffffu);
        if (!start) continue;
        int kb = csr_ptr[node], ke = csr_ptr[node + 1];
        int first = csr_ent[kb] / nv, last = csr_ent[ke - 1] / nv;
        bool earlier = first < e0;
        bool nonowner = last >= e1;
        sfix[runid[i]] = (earlier && !nonowner) ? 1 : 0;
        if (mode == 0) {
            if (earlier && !nonowner) atomicMin(&s_mindep, block_of(first, blk_elem, nb));
        } else {
            int o = blk_occ[b] + runid[i];
            occ_node[o] = node | (nonowner ? OCC_NONOWNER : 0) | (earlier && !nonowner ? OCC_EARLIER : 0);
            occ_ent_ptr[o] = e0 * nv + i;
            // rank of this block among the node's blocks = distinct blocks with elements < e0
            int rank = 0, lastb = -1;
            for (int k = kb; k < ke; ++k) {
                int f = csr_ent[k] / nv;
                if (f >= e0) break;
                int bb = block_of(f, blk_elem, nb);
                if (bb != lastb) { ++rank; lastb = bb; }
            }
            node_occ[node_occ_ptr[node] + rank] = o;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int nf = 0;
        for (int r2 = 0; r2 < n_occ_b; ++r2) {
            if (!sfix[r2]) continue;
            if (mode == 1) fix_occ[blk_fix[b] + nf] = blk_occ[b] + r2;
            ++nf;
        }
        if (mode == 0) {
            occ_cnt[b] = n_occ_b;
            fix_cnt[b] = nf;
            min_dep[b] = s_mindep;
        }
    }
}

// fix-up source lists: for each fix entry (owned node with earlier partials) all occurrences
// of its node in ascending block order (the last one is the owner's own segment)
__global__ void k_fix_count(int n_fix, const int32_t* __restrict__ fix_occ, const int32_t* __restrict__ occ_node,
                            const int32_t* __restrict__ node_occ_ptr, int32_t* cnt, int32_t* fix_node) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n_fix) return;
    const int node = occ_node[fix_occ[f]] & OCC_NODE_MASK;
    fix_node[f] = node;
    cnt[f] = node_occ_ptr[node + 1] - node_occ_ptr[node];
}

__global__ void k_fix_fill(int n_fix, const int32_t* __restrict__ fix_node, const int32_t* __restrict__ node_occ_ptr,
                           const int32_t* __restrict__ node_occ, const int32_t* __restrict__ fix_src_ptr,
                           int32_t* fix_src, int32_t* occ_seg) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n_fix) return;
    const int node = fix_node[f];
    const int k0 = node_occ_ptr[node], k1 = node_occ_ptr[node + 1];
    for (int k = k0; k < k1; ++k) {
        fix_src[fix_src_ptr[f] + (k - k0)] = node_occ[k];
        occ_seg[node_occ[k]] = fix_src_ptr[f] + (k - k0);
    }
}

// packed block records (see RecLayout): grid = blocks
template <int D, class T>
__global__ void k_pack_records(int E, const int32_t* __restrict__ blk_elem, const int32_t* __restrict__ blk_occ,
                               const int32_t* __restrict__ conn, const T* __restrict__ grad,
                               const T* __restrict__ vol, const int32_t* __restrict__ occ_node,
                               const int32_t* __restrict__ occ_ent_ptr, const uint16_t* __restrict__ loc_ent,
                               const int32_t* __restrict__ occ_seg, const int32_t* __restrict__ perm,
                               unsigned char* recs, RecLayout L) {
    // conn (and every index here) is in plan positions; grad / vol are read at the input
    // element perm[position] (identity when perm is null), whose id the record keeps (eid)
    constexpr int NV = D + 1;
    const int b = blockIdx.x;
    const int e0 = blk_elem[b], ne = blk_elem[b + 1] - e0;
    const int o0 = blk_occ[b], no = blk_occ[b + 1] - o0;
    unsigned char* r = recs + (size_t)b * L.bytes;
    int32_t* rc = reinterpret_cast<int32_t*>(r + L.conn);
    T* rg = reinterpret_cast<T*>(r + L.g);
    T* rv = reinterpret_cast<T*>(r + L.vol);
    int32_t* ron = reinterpret_cast<int32_t*>(r + L.occ_node);
    uint16_t* roe = reinterpret_cast<uint16_t*>(r + L.occ_ent);
    uint16_t* rle = reinterpret_cast<uint16_t*>(r + L.loc_ent);
    int32_t* rid = reinterpret_cast<int32_t*>(r + L.eid);
    for (int el = threadIdx.x; el < L.eb; el += blockDim.x) {
        const bool in = el < ne;
        const int src = !in ? 0 : (perm ? perm[e0 + el] : e0 + el);
#pragma unroll
        for (int a = 0; a < NV; ++a) rc[el * NV + a] = in ? conn[(int64_t)(e0 + el) * NV + a] : 0;
#pragma unroll
        for (int k = 0; k < D * D; ++k) rg[k * L.eb + el] = in ? grad[(int64_t)k * E + src] : T(0);
        rv[el] = in ? vol[src] : T(0);
        if (perm) rid[el] = in ? src : 0;
    }
    for (int i = threadIdx.x; i < L.ocap; i += blockDim.x) ron[i] = i < no ? occ_node[o0 + i] : 0;
    int32_t* ros = reinterpret_cast<int32_t*>(r + L.occ_seg);
    for (int i = threadIdx.x; i < L.ocap; i += blockDim.x) ros[i] = i < no ? occ_seg[o0 + i] : -1;
    for (int i = threadIdx.x; i <= L.ocap; i += blockDim.x)
        roe[i] = (uint16_t)(i <= no ? occ_ent_ptr[o0 + i] - NV * e0 : NV * ne);
    uint16_t* rep = reinterpret_cast<uint16_t*>(r + L.ent_pos);
    for (int k = threadIdx.x; k < NV * L.eb; k += blockDim.x) {
        // the record keeps each entry's force-buffer slot a * EB + el (element-major buffer)
        // rather than the plan's el * (d+1) + a, so phase 2 needs no division
        if (k < NV * ne) {
            const int j = loc_ent[(int64_t)NV * e0 + k];
            rle[k] = (uint16_t)((j % NV) * L.eb + j / NV);
        } else {
            rle[k] = 0;
        }
        if (k < NV * ne) rep[loc_ent[(int64_t)NV * e0 + k]] = (uint16_t)k;   // a permutation of [0, NV ne)
        else rep[k] = (uint16_t)k;
    }
    // local occurrence index of each element vertex: binary search in the block's sorted nodes
    uint16_t* rlc = reinterpret_cast<uint16_t*>(r + L.lconn);
    for (int k = threadIdx.x; k < NV * L.eb; k += blockDim.x) {
        uint16_t idx = 0;
        if (k < NV * ne) {
            const int node = conn[(int64_t)NV * e0 + k];
            int lo = 0, hi = no - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if ((occ_node[o0 + mid] & OCC_NODE_MASK) < node) lo = mid + 1;
                else hi = mid;
            }
            idx = (uint16_t)lo;
        }
        rlc[k] = idx;
    }
    // phase-2 order: occurrences by descending entry count, ties by index (a permutation)
    uint16_t* rop = reinterpret_cast<uint16_t*>(r + L.occ_perm);
    for (int i = threadIdx.x; i < L.ocap; i += blockDim.x) {
        if (i >= no) {
            rop[i] = (uint16_t)i;
            continue;
        }
        const int ci = occ_ent_ptr[o0 + i + 1] - occ_ent_ptr[o0 + i];
        int rank = 0;
        for (int j = 0; j < no; ++j) {
            const int cj = occ_ent_ptr[o0 + j + 1] - occ_ent_ptr[o0 + j];
            rank += (cj > ci || (cj == ci && j < i)) ? 1 : 0;
        }
        rop[rank] = (uint16_t)i;
    }
}

// ------------------------------------------------------------------ host driver
namespace {

struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

pfem_status exclusive_scan_i32(const int32_t* in, int32_t* out, int n, cudaStream_t s) {
    size_t tb = 0;
    PFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s));
    DevBuf tmp;
    tmp.s = s;
    PFEM_CUDA_TRY(cudaMallocAsync(&tmp.p, tb, s));
    PFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, s));
    count_launch();
    return PFEM_OK;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

pfem_status quad_prepare_geometry(const pfem_mesh* m, Plan* P, cudaStream_t s);   // quad.cu
void release_impl(pfem_mesh* m);

pfem_status prepare_impl(pfem_mesh* m, cudaStream_t s) {
    const bool quad = m->elem_type != PFEM_ELEM_SIMPLEX;
    const int D = m->dim, N = m->n_nodes, E = m->n_elems;
    const int nv = quad ? (m->elem_type == PFEM_ELEM_Q4 ? 4 : 8) : D + 1;
    const int K = m->n_parts;
    // ---------------- validation of connectivity
    DevBuf scratch;
    scratch.s = s;
    const size_t n_int_scratch = 8 + (size_t)std::max(N + 1, m->max_colours + 1);
    PFEM_CUDA_TRY(cudaMallocAsync(&scratch.p, sizeof(int32_t) * n_int_scratch, s));
    int32_t* sc = (int32_t*)scratch.p;            // [0]=bad conn [1]=n_neg [2]=degenerate [3]=overflow [4]=maxc [5]=ticket
    int32_t* cnt = sc + 8;                        // [N+1]
    int32_t init[8] = {INT32_MAX, 0, INT32_MAX, INT32_MAX, -1, 0, 0, 0};
    PFEM_CUDA_TRY(cudaMemcpyAsync(sc, init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_check_conn<<<nblk((int64_t)E * nv, 256), 256, 0, s>>>(nv, E, N, m->conn, sc + 0);
    PFEM_LAUNCH_CHECK("k_check_conn");
    // ---------------- K1 geometry (quadrilaterals: per Gauss point, after the CSR)
    if (quad) {
    } else if (D == 2) {
        if (m->dtype == PFEM_F32)
            k_geometry<2, float><<<nblk(E, 256), 256, 0, s>>>(E, m->coords, m->conn, (float*)m->grad,
                                                                (float*)m->vol, sc + 1, sc + 2);
        else
            k_geometry<2, double><<<nblk(E, 256), 256, 0, s>>>(E, m->coords, m->conn, (double*)m->grad,
                                                                 (double*)m->vol, sc + 1, sc + 2);
    } else {
        if (m->dtype == PFEM_F32)
            k_geometry<3, float><<<nblk(E, 256), 256, 0, s>>>(E, m->coords, m->conn, (float*)m->grad,
                                                                (float*)m->vol, sc + 1, sc + 2);
        else
            k_geometry<3, double><<<nblk(E, 256), 256, 0, s>>>(E, m->coords, m->conn, (double*)m->grad,
                                                                 (double*)m->vol, sc + 1, sc + 2);
    }
    PFEM_LAUNCH_CHECK("k_geometry");
    int32_t h[8];
    PFEM_CUDA_TRY(cudaMemcpyAsync(h, sc, sizeof(h), cudaMemcpyDeviceToHost, s));
    PFEM_CUDA_TRY(cudaStreamSynchronize(s));
    if (h[0] != INT32_MAX) {
        set_error("conn: node id out of range [0, n_nodes)", h[0]);
        return PFEM_ERR_ARG;
    }
    if (h[2] != INT32_MAX) {
        set_error("degenerate element (|det J| <= 64 eps prod |edges|)", h[2]);
        return PFEM_ERR_DEGENERATE;
    }
    m->n_negative = h[1];
    // ---------------- K2 CSR
    const int64_t nent = (int64_t)E * nv;
    PFEM_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (N + 1), s));
    k_count<<<nblk(nent, 256), 256, 0, s>>>(nent, m->conn, cnt);
    PFEM_LAUNCH_CHECK("k_count");
    {
        pfem_status st = exclusive_scan_i32(cnt, m->csr_ptr, N + 1, s);
        if (st != PFEM_OK) return st;
    }
    PFEM_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (N + 1), s));
    k_csr_fill<<<nblk(nent, 256), 256, 0, s>>>(nent, m->conn, m->csr_ptr, cnt, m->csr_ent);
    PFEM_LAUNCH_CHECK("k_csr_fill");
    k_csr_sort_rows<<<nblk(N, 128), 128, 0, s>>>(N, m->csr_ptr, m->csr_ent);
    PFEM_LAUNCH_CHECK("k_csr_sort_rows");
    // ---------------- K3 colouring
    PFEM_CUDA_TRY(cudaMemsetAsync(m->colour, 0xff, sizeof(int32_t) * E, s));
    {
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        k_colour_greedy<<<nsm * 8, 256, 0, s>>>(nv, E, m->conn, m->csr_ptr, m->csr_ent, m->colour, sc + 5,
                                                  m->max_colours, sc + 3);
        PFEM_LAUNCH_CHECK("k_colour_greedy");
    }
    PFEM_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (m->max_colours + 1), s));
    k_colour_hist<<<nblk(E, 256), 256, 0, s>>>(E, m->colour, cnt, sc + 4);
    PFEM_LAUNCH_CHECK("k_colour_hist");
    PFEM_CUDA_TRY(cudaMemcpyAsync(h, sc, sizeof(h), cudaMemcpyDeviceToHost, s));
    PFEM_CUDA_TRY(cudaStreamSynchronize(s));
    if (h[3] != INT32_MAX) {
        set_error("more colours than max_colours", h[3]);
        return PFEM_ERR_CAPACITY;
    }
    m->n_colours = h[4] + 1;
    k_colour_ptr<<<1, 32, 0, s>>>(m->n_colours, cnt, m->colour_ptr);
    PFEM_LAUNCH_CHECK("k_colour_ptr");
    {
        // stable radix sort of (colour, element) pairs -> colour_elems
        DevBuf tmp;
        tmp.s = s;
        int end_bit = 1;
        while ((1 << end_bit) <= m->n_colours) ++end_bit;
        size_t tb = 0;
        int32_t* keys_out = nullptr;
        int32_t* vals_in = nullptr;
        PFEM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, m->colour, keys_out, vals_in,
                                                      m->colour_elems, E, 0, end_bit, s));
        size_t extra = align_up(sizeof(int32_t) * (size_t)E, 256);
        PFEM_CUDA_TRY(cudaMallocAsync(&tmp.p, tb + 2 * extra, s));
        keys_out = (int32_t*)tmp.p;
        vals_in = (int32_t*)((char*)tmp.p + extra);
        void* t2 = (char*)tmp.p + 2 * extra;
        k_iota<<<nblk(E, 256), 256, 0, s>>>(E, vals_in);
        PFEM_LAUNCH_CHECK("k_iota");
        PFEM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(t2, tb, m->colour, keys_out, vals_in,
                                                      m->colour_elems, E, 0, end_bit, s));
        count_launch();
    }
    // ---------------- quadrilaterals: Gauss-point geometry and CSR entry positions, no block plan
    if (quad) {
        Plan* P = new Plan();
        static std::atomic<uint64_t> quad_serial{1ull << 40};
        P->serial = ++quad_serial;
        P->dim = D; P->n_nodes = N; P->n_elems = E; P->n_parts = K;
        P->elem_type = m->elem_type;
        P->nv = nv;
        std::vector<int32_t> qpe{0, E}, qpn{0, N};
        if (K > 1) {
            qpe.resize(K + 1);
            qpn.resize(K + 1);
            PFEM_CUDA_TRY(cudaMemcpyAsync(qpe.data(), m->part_elem, sizeof(int32_t) * (K + 1), cudaMemcpyDeviceToHost, s));
            PFEM_CUDA_TRY(cudaMemcpyAsync(qpn.data(), m->part_node, sizeof(int32_t) * (K + 1), cudaMemcpyDeviceToHost, s));
        }
        cudaError_t ce = cudaMallocAsync(&P->pool, 2 * align_up(sizeof(int32_t) * (K + 1), 256), s);
        if (ce != cudaSuccess) { delete P; return cuda_status(ce, "plan alloc"); }
        P->part_elem = (int32_t*)P->pool;
        P->part_node = (int32_t*)((char*)P->pool + align_up(sizeof(int32_t) * (K + 1), 256));
        PFEM_CUDA_TRY(cudaMemcpyAsync(P->part_elem, qpe.data(), sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, s));
        PFEM_CUDA_TRY(cudaMemcpyAsync(P->part_node, qpn.data(), sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, s));
        P->colour_ptr_host.resize(m->n_colours + 1);
        PFEM_CUDA_TRY(cudaMemcpyAsync(P->colour_ptr_host.data(), m->colour_ptr, sizeof(int32_t) * (m->n_colours + 1),
                                      cudaMemcpyDeviceToHost, s));
        m->plan = reinterpret_cast<pfem_plan*>(P);   // released by release_impl on failure below
        const pfem_status st = quad_prepare_geometry(m, P, s);
        if (st != PFEM_OK) {
            release_impl(m);
            return st;
        }
        m->n_negative = 0;
        m->n_blocks = 0;
        m->n_occ = 0;
        return PFEM_OK;
    }
    // ---------------- plan: element blocks (host bookkeeping on the part offsets)
    std::vector<int32_t> pe(K + 1), pn(K + 1);
    if (K == 1 || !m->part_elem) {
        pe = {0, E};
        pn = {0, N};
    } else {
        PFEM_CUDA_TRY(cudaMemcpyAsync(pe.data(), m->part_elem, sizeof(int32_t) * (K + 1), cudaMemcpyDeviceToHost, s));
        PFEM_CUDA_TRY(cudaMemcpyAsync(pn.data(), m->part_node, sizeof(int32_t) * (K + 1), cudaMemcpyDeviceToHost, s));
        PFEM_CUDA_TRY(cudaStreamSynchronize(s));
        if (pe[0] != 0 || pe[K] != E || pn[0] != 0 || pn[K] != N) {
            set_error("part offsets must start at 0 and end at n_elems / n_nodes");
            return PFEM_ERR_ARG;
        }
        for (int k = 0; k < K; ++k)
            if (pe[k + 1] < pe[k] || pn[k + 1] < pn[k]) {
                set_error("part offsets must be non-decreasing", k);
                return PFEM_ERR_ARG;
            }
    }
    // block capacity = the CSR kernel's compile-time EB (assemble.cuh EbOf): 256 T4 / 512 T3
    // (a larger block_elems, up to PLAN_MAX_KEYS / (d+1), is served by the direct kernel form)
    // defaults: the staged kernel's capacity (T4 256, T3 512); fp64 T4 plans 384 — their calls
    // are single-sample solves (K.v in CG / Newton) served by the direct form, where larger
    // blocks mean fewer multi-block nodes (measured on config 4: 131 -> 123 us)
    const int eb_default = D == 3 ? (m->dtype == PFEM_F64 ? 384 : 256) : 512;
    int eb = m->block_elems > 0 ? m->block_elems : eb_default;
    eb = std::min(eb, PLAN_MAX_KEYS / nv);
    const int eb_cap = std::max(eb, eb_default);
    std::vector<int32_t> blk_elem{0}, part_blk{0};
    for (int k = 0; k < K; ++k) {
        int n = pe[k + 1] - pe[k];
        int nbk = (n + eb - 1) / eb;
        for (int i = 1; i <= nbk; ++i) blk_elem.push_back(pe[k] + (int)((int64_t)n * i / nbk));
        part_blk.push_back((int)blk_elem.size() - 1);
    }
    const int nb = (int)blk_elem.size() - 1;
    int eb_max = 0;
    for (int b = 0; b < nb; ++b) eb_max = std::max(eb_max, blk_elem[b + 1] - blk_elem[b]);

    // reduction chunks: <= CHUNK consecutive blocks inside one part
    std::vector<int32_t> blk_chunk(nb), chunk_blk{0}, part_chunk{0};
    for (int k = 0; k < K; ++k) {
        for (int b0 = part_blk[k]; b0 < part_blk[k + 1]; b0 += CHUNK_BLOCKS) {
            int b1 = std::min(part_blk[k + 1], b0 + CHUNK_BLOCKS);
            for (int b = b0; b < b1; ++b) blk_chunk[b] = (int)chunk_blk.size() - 1;
            chunk_blk.push_back(b1);
        }
        part_chunk.push_back((int)chunk_blk.size() - 1);
    }
    const int nch = (int)chunk_blk.size() - 1;

    Plan* P = new Plan();
    static std::atomic<uint64_t> plan_serial{0};
    P->serial = ++plan_serial;
    P->dim = D; P->n_nodes = N; P->n_elems = E; P->n_parts = K;
    P->n_blocks = nb; P->eb_max = eb_max; P->n_chunks = nch;
    // first allocation: everything whose size is known now
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t at = o; o += align_up(bytes, 256); return at; };
    size_t o_be = take(sizeof(int32_t) * (nb + 1)), o_bo = take(sizeof(int32_t) * (nb + 1)),
           o_md = take(sizeof(int32_t) * (nb + 1)), o_pb = take(sizeof(int32_t) * (K + 1)),
           o_pn = take(sizeof(int32_t) * (K + 1)), o_pe = take(sizeof(int32_t) * (K + 1)),
           o_bc = take(sizeof(int32_t) * (nb + 1)), o_cb = take(sizeof(int32_t) * (nch + 1)),
           o_pc = take(sizeof(int32_t) * (K + 1)), o_le = take(sizeof(uint16_t) * (size_t)nent),
           o_np = take(sizeof(int32_t) * ((size_t)N + 1)), o_cnt = take(sizeof(int32_t) * (nb + 1)),
           o_fc = take(sizeof(int32_t) * (nb + 1)), o_bf = take(sizeof(int32_t) * (nb + 1));
    size_t fixed = o;
    void* pool1 = nullptr;
    cudaError_t ce = cudaMallocAsync(&pool1, fixed, s);
    if (ce != cudaSuccess) { delete P; return cuda_status(ce, "plan alloc"); }
    auto bind = [&](char* pb) {
        P->blk_elem = (int32_t*)(pb + o_be);
        P->blk_occ = (int32_t*)(pb + o_bo);
        P->blk_min_dep = (int32_t*)(pb + o_md);
        P->part_blk = (int32_t*)(pb + o_pb);
        P->part_node = (int32_t*)(pb + o_pn);
        P->part_elem = (int32_t*)(pb + o_pe);
        P->blk_chunk = (int32_t*)(pb + o_bc);
        P->chunk_blk = (int32_t*)(pb + o_cb);
        P->part_chunk = (int32_t*)(pb + o_pc);
        P->loc_ent = (uint16_t*)(pb + o_le);
        P->node_occ_ptr = (int32_t*)(pb + o_np);
        P->blk_fix = (int32_t*)(pb + o_bf);
    };
    bind((char*)pool1);
    int32_t* occ_cnt = (int32_t*)((char*)pool1 + o_cnt);
    int32_t* fix_cnt = (int32_t*)((char*)pool1 + o_fc);
    P->pool = pool1;
    auto fail = [&](pfem_status st) {
        cudaFreeAsync(P->pool, s);
        if (P->pool_perm) cudaFreeAsync(P->pool_perm, s);
        delete P;
        return st;
    };
#define PLAN_TRY(expr) do { cudaError_t _e = (expr); if (_e != cudaSuccess) return fail(cuda_status(_e, #expr)); } while (0)
    PLAN_TRY(cudaMemcpyAsync(P->blk_elem, blk_elem.data(), sizeof(int32_t) * (nb + 1), cudaMemcpyHostToDevice, s));
    PLAN_TRY(cudaMemcpyAsync(P->part_blk, part_blk.data(), sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, s));
    PLAN_TRY(cudaMemcpyAsync(P->part_node, pn.data(), sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, s));
    PLAN_TRY(cudaMemcpyAsync(P->part_elem, pe.data(), sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, s));
    PLAN_TRY(cudaMemcpyAsync(P->blk_chunk, blk_chunk.data(), sizeof(int32_t) * nb, cudaMemcpyHostToDevice, s));
    PLAN_TRY(cudaMemcpyAsync(P->chunk_blk, chunk_blk.data(), sizeof(int32_t) * (nch + 1), cudaMemcpyHostToDevice, s));
    PLAN_TRY(cudaMemcpyAsync(P->part_chunk, part_chunk.data(), sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, s));
    P->colour_ptr_host.resize(m->n_colours + 1);
    PLAN_TRY(cudaMemcpyAsync(P->colour_ptr_host.data(), m->colour_ptr, sizeof(int32_t) * (m->n_colours + 1),
                             cudaMemcpyDeviceToHost, s));
    // ---------------- element order of the plan (positions)
    const int32_t* pconn = m->conn;
    const int32_t* pptr = m->csr_ptr;
    const int32_t* pent = m->csr_ent;
    if (m->elem_order != PFEM_ORDER_INPUT && E > 0) {
        {
            const size_t a_perm = align_up(sizeof(int32_t) * (size_t)E, 256);
            const size_t a_conn = align_up(sizeof(int32_t) * (size_t)E * nv, 256);
            const size_t a_ptr = align_up(sizeof(int32_t) * ((size_t)N + 1), 256);
            void* pp = nullptr;
            PLAN_TRY(cudaMallocAsync(&pp, a_perm + 2 * a_conn + a_ptr, s));
            P->pool_perm = pp;
            P->elem_perm = (int32_t*)pp;
            P->conn_p = (int32_t*)((char*)pp + a_perm);
            P->csr_ent_p = (int32_t*)((char*)pp + a_perm + a_conn);
            P->csr_ptr_p = (int32_t*)((char*)pp + a_perm + 2 * a_conn);
        }
        {
            // Morton keys of the centroids (part id in the high word), stable radix sort
            DevBuf tmp;
            tmp.s = s;
            const size_t a_key = align_up(sizeof(unsigned long long) * (size_t)E, 256);
            const size_t a_val = align_up(sizeof(int32_t) * (size_t)E, 256);
            int end_bit = 32;
            while ((1ll << (end_bit - 32)) < K) ++end_bit;
            size_t tb = 0;
            PLAN_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, (unsigned long long*)nullptr,
                                                     (unsigned long long*)nullptr, (int32_t*)nullptr,
                                                     P->elem_perm, E, 0, end_bit, s));
            PLAN_TRY(cudaMallocAsync(&tmp.p, 2 * a_key + a_val + 256 + tb, s));
            unsigned long long* kin = (unsigned long long*)tmp.p;
            unsigned long long* kout = (unsigned long long*)((char*)tmp.p + a_key);
            int32_t* vin = (int32_t*)((char*)tmp.p + 2 * a_key);
            unsigned long long* bb = (unsigned long long*)((char*)tmp.p + 2 * a_key + a_val);
            void* t2 = (char*)tmp.p + 2 * a_key + a_val + 256;
            unsigned long long bb0[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
            unsigned long long bbi[6];
            for (int j = 0; j < D; ++j) { bbi[j] = bb0[0]; bbi[D + j] = 0ull; }
            PLAN_TRY(cudaMemcpyAsync(bb, bbi, sizeof(unsigned long long) * 2 * D, cudaMemcpyHostToDevice, s));
            k_bbox<<<std::max(1u, std::min(nblk(N, 256), 1184u)), 256, 0, s>>>(N, D, m->coords, bb);
            count_launch();
            k_morton_keys<<<nblk(E, 256), 256, 0, s>>>(E, D, K, m->coords, m->conn, P->part_elem, bb, kin, vin);
            count_launch();
            PLAN_TRY(cudaGetLastError());
            PLAN_TRY(cub::DeviceRadixSort::SortPairs(t2, tb, kin, kout, vin, P->elem_perm, E, 0, end_bit, s));
            count_launch();
            PLAN_TRY(cudaStreamSynchronize(s));   // tmp is released at scope end
        }
        k_gather_conn<<<nblk((int64_t)E * nv, 256), 256, 0, s>>>(E, nv, P->elem_perm, m->conn, P->conn_p);
        count_launch();
        // node -> (position, slot) CSR of the ordered connectivity
        PLAN_TRY(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (N + 1), s));
        k_count<<<nblk(nent, 256), 256, 0, s>>>(nent, P->conn_p, cnt);
        count_launch();
        {
            pfem_status st = exclusive_scan_i32(cnt, P->csr_ptr_p, N + 1, s);
            if (st != PFEM_OK) return fail(st);
        }
        PLAN_TRY(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (N + 1), s));
        k_csr_fill<<<nblk(nent, 256), 256, 0, s>>>(nent, P->conn_p, P->csr_ptr_p, cnt, P->csr_ent_p);
        count_launch();
        k_csr_sort_rows<<<nblk(N, 128), 128, 0, s>>>(N, P->csr_ptr_p, P->csr_ent_p);
        count_launch();
        PLAN_TRY(cudaGetLastError());
        if (m->elem_order == PFEM_ORDER_AUTO) {
            // keep the order with fewer (block, node) occurrences (block-local sort counts)
            int32_t tot[2] = {0, 0};
            for (int v = 0; v < 2; ++v) {
                k_block_build<<<nb, PLAN_THREADS, 0, s>>>(0, nv, nb, P->blk_elem, v ? P->conn_p : m->conn,
                                                          v ? P->csr_ptr_p : m->csr_ptr, v ? P->csr_ent_p : m->csr_ent,
                                                          occ_cnt, fix_cnt, P->blk_min_dep, nullptr, nullptr, nullptr,
                                                          nullptr, nullptr, nullptr, nullptr, nullptr);
                count_launch();
                PLAN_TRY(cudaGetLastError());
                PLAN_TRY(cudaMemsetAsync(occ_cnt + nb, 0, sizeof(int32_t), s));
                pfem_status st = exclusive_scan_i32(occ_cnt, P->blk_occ, nb + 1, s);
                if (st != PFEM_OK) return fail(st);
                PLAN_TRY(cudaMemcpyAsync(&tot[v], P->blk_occ + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
                PLAN_TRY(cudaStreamSynchronize(s));
            }
            if (tot[1] >= tot[0]) {
                PLAN_TRY(cudaFreeAsync(P->pool_perm, s));
                P->pool_perm = nullptr;
                P->elem_perm = P->conn_p = P->csr_ptr_p = P->csr_ent_p = nullptr;
            }
        }
    }
    if (P->elem_perm) {
        pconn = P->conn_p;
        pptr = P->csr_ptr_p;
        pent = P->csr_ent_p;
    }
    P->elem_order = P->elem_perm ? 1 : 0;
    // node-major occurrence counts -> node_occ_ptr
    k_node_occ_count<<<nblk(N, 256), 256, 0, s>>>(N, nv, pptr, pent, P->blk_elem, nb, cnt);
    count_launch();
    PLAN_TRY(cudaGetLastError());
    {
        pfem_status st = exclusive_scan_i32(cnt, P->node_occ_ptr, N + 1, s);
        if (st != PFEM_OK) return fail(st);
    }
    k_block_build<<<nb, PLAN_THREADS, 0, s>>>(0, nv, nb, P->blk_elem, pconn, pptr, pent,
                                              occ_cnt, fix_cnt, P->blk_min_dep, nullptr, nullptr, nullptr,
                                              nullptr, nullptr, nullptr, nullptr, nullptr);
    count_launch();
    PLAN_TRY(cudaGetLastError());
    PLAN_TRY(cudaMemsetAsync(occ_cnt + nb, 0, sizeof(int32_t), s));
    PLAN_TRY(cudaMemsetAsync(fix_cnt + nb, 0, sizeof(int32_t), s));
    {
        pfem_status st = exclusive_scan_i32(occ_cnt, P->blk_occ, nb + 1, s);
        if (st != PFEM_OK) return fail(st);
        st = exclusive_scan_i32(fix_cnt, P->blk_fix, nb + 1, s);
        if (st != PFEM_OK) return fail(st);
    }
    int32_t n_occ = 0, n_fix = 0;
    PLAN_TRY(cudaMemcpyAsync(&n_occ, P->blk_occ + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    PLAN_TRY(cudaMemcpyAsync(&n_fix, P->blk_fix + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    PLAN_TRY(cudaStreamSynchronize(s));
    P->n_occ = n_occ;
    P->n_fix = n_fix;
    // second allocation: occurrence arrays
    size_t o2 = 0;
    auto take2 = [&](size_t bytes) { size_t at = o2; o2 += align_up(bytes, 256); return at; };
    size_t q_on = take2(sizeof(int32_t) * (size_t)n_occ), q_oe = take2(sizeof(int32_t) * ((size_t)n_occ + 1)),
           q_no = take2(sizeof(int32_t) * (size_t)n_occ), q_fo = take2(sizeof(int32_t) * ((size_t)n_fix + 1));
    // grow the pool: allocate a new pool of fixed + o2 and copy the fixed part
    void* pool2 = nullptr;
    PLAN_TRY(cudaMallocAsync(&pool2, fixed + o2, s));
    PLAN_TRY(cudaMemcpyAsync(pool2, pool1, fixed, cudaMemcpyDeviceToDevice, s));
    PLAN_TRY(cudaFreeAsync(pool1, s));
    P->pool = pool2;
    char* pb = (char*)pool2;
    bind(pb);
    P->occ_node = (int32_t*)(pb + fixed + q_on);
    P->occ_ent_ptr = (int32_t*)(pb + fixed + q_oe);
    P->node_occ = (int32_t*)(pb + fixed + q_no);
    P->fix_occ = (int32_t*)(pb + fixed + q_fo);
    occ_cnt = (int32_t*)(pb + o_cnt);
    k_block_build<<<nb, PLAN_THREADS, 0, s>>>(1, nv, nb, P->blk_elem, pconn, pptr, pent,
                                              nullptr, nullptr, nullptr, P->blk_occ, P->occ_node, P->occ_ent_ptr,
                                              P->loc_ent, P->node_occ_ptr, P->node_occ, P->blk_fix, P->fix_occ);
    count_launch();
    PLAN_TRY(cudaGetLastError());
    int32_t tail = (int32_t)nent;
    PLAN_TRY(cudaMemcpyAsync(P->occ_ent_ptr + n_occ, &tail, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    // fix-up source lists (third allocation)
    {
        const int nf = std::max(1, n_fix);
        size_t o3 = 0;
        auto take3 = [&](size_t bytes) { size_t at = o3; o3 += align_up(bytes, 256); return at; };
        size_t r_ptr = take3(sizeof(int32_t) * ((size_t)nf + 1)), r_node = take3(sizeof(int32_t) * (size_t)nf),
               r_cnt = take3(sizeof(int32_t) * ((size_t)nf + 1));
        void* pool3 = nullptr;
        PLAN_TRY(cudaMallocAsync(&pool3, o3, s));
        P->pool_fix = pool3;
        P->fix_src_ptr = (int32_t*)((char*)pool3 + r_ptr);
        P->fix_node = (int32_t*)((char*)pool3 + r_node);
        int32_t* fcnt = (int32_t*)((char*)pool3 + r_cnt);
        PLAN_TRY(cudaMemsetAsync(fcnt, 0, sizeof(int32_t) * ((size_t)nf + 1), s));
        if (n_fix > 0) {
            k_fix_count<<<nblk(n_fix, 256), 256, 0, s>>>(n_fix, P->fix_occ, P->occ_node, P->node_occ_ptr, fcnt, P->fix_node);
            count_launch();
            PLAN_TRY(cudaGetLastError());
        }
        pfem_status st = exclusive_scan_i32(fcnt, P->fix_src_ptr, n_fix + 1, s);
        if (st != PFEM_OK) return fail(st);
        int32_t n_src = 0;
        PLAN_TRY(cudaMemcpyAsync(&n_src, P->fix_src_ptr + n_fix, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        PLAN_TRY(cudaStreamSynchronize(s));
        void* pool4 = nullptr;
        const size_t src_bytes = align_up(sizeof(int32_t) * (size_t)std::max(1, n_src), 256);
        PLAN_TRY(cudaMallocAsync(&pool4, src_bytes + sizeof(int32_t) * (size_t)std::max(1, n_occ), s));
        P->pool_src = pool4;
        P->fix_src = (int32_t*)pool4;
        P->occ_seg = (int32_t*)((char*)pool4 + src_bytes);
        P->n_seg = n_src;
        PLAN_TRY(cudaMemsetAsync(P->occ_seg, 0xff, sizeof(int32_t) * (size_t)std::max(1, n_occ), s));
        if (n_fix > 0) {
            k_fix_fill<<<nblk(n_fix, 256), 256, 0, s>>>(n_fix, P->fix_node, P->node_occ_ptr, P->node_occ,
                                                         P->fix_src_ptr, P->fix_src, P->occ_seg);
            count_launch();
            PLAN_TRY(cudaGetLastError());
        }
    }
    // packed block records (one TMA bulk copy per block in the CSR kernel)
    {
        std::vector<int32_t> bo(nb + 1);
        PLAN_TRY(cudaMemcpyAsync(bo.data(), P->blk_occ, sizeof(int32_t) * (nb + 1), cudaMemcpyDeviceToHost, s));
        PLAN_TRY(cudaStreamSynchronize(s));
        int ocap = 8;
        for (int b = 0; b < nb; ++b) ocap = std::max(ocap, bo[b + 1] - bo[b]);
        ocap = (ocap + 7) / 8 * 8;
        const size_t ts = m->dtype == PFEM_F64 ? 8 : 4;
        P->rec = rec_layout(D, ts, eb_cap, ocap, P->elem_perm != nullptr);
        void* pr = nullptr;
        PLAN_TRY(cudaMallocAsync(&pr, (size_t)P->rec.bytes * nb, s));
        P->pool_rec = pr;
        P->recs = (unsigned char*)pr;
        if (D == 2) {
            if (ts == 4)
                k_pack_records<2, float><<<nb, 256, 0, s>>>(E, P->blk_elem, P->blk_occ, pconn, (const float*)m->grad,
                    (const float*)m->vol, P->occ_node, P->occ_ent_ptr, P->loc_ent, P->occ_seg, P->elem_perm, P->recs, P->rec);
            else
                k_pack_records<2, double><<<nb, 256, 0, s>>>(E, P->blk_elem, P->blk_occ, pconn, (const double*)m->grad,
                    (const double*)m->vol, P->occ_node, P->occ_ent_ptr, P->loc_ent, P->occ_seg, P->elem_perm, P->recs, P->rec);
        } else {
            if (ts == 4)
                k_pack_records<3, float><<<nb, 256, 0, s>>>(E, P->blk_elem, P->blk_occ, pconn, (const float*)m->grad,
                    (const float*)m->vol, P->occ_node, P->occ_ent_ptr, P->loc_ent, P->occ_seg, P->elem_perm, P->recs, P->rec);
            else
                k_pack_records<3, double><<<nb, 256, 0, s>>>(E, P->blk_elem, P->blk_occ, pconn, (const double*)m->grad,
                    (const double*)m->vol, P->occ_node, P->occ_ent_ptr, P->loc_ent, P->occ_seg, P->elem_perm, P->recs, P->rec);
        }
        count_launch();
        PLAN_TRY(cudaGetLastError());
    }
    PLAN_TRY(cudaStreamSynchronize(s));
#undef PLAN_TRY
    m->n_blocks = nb;
    m->n_occ = n_occ;
    m->plan = reinterpret_cast<pfem_plan*>(P);
    return PFEM_OK;
}

void release_impl(pfem_mesh* m) {
    if (!m || !m->plan) return;
    Plan* P = reinterpret_cast<Plan*>(m->plan);
    if (P->pool) cudaFree(P->pool);
    if (P->pool_fix) cudaFree(P->pool_fix);
    if (P->pool_src) cudaFree(P->pool_src);
    if (P->pool_rec) cudaFree(P->pool_rec);
    if (P->pool_perm) cudaFree(P->pool_perm);
    if (P->pool_quad) cudaFree(P->pool_quad);
    delete P;
    m->plan = nullptr;
}

}  // namespace pfem

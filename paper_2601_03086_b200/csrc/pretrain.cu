// pretrain.cu — the pretraining-loss epilogue of the hot path:
//   u = phi (.) H                     hard-BC ansatz u = (x/L) (.) H_theta (R28)
//   Pi_{s,k} = W_{s,k}(u) - f_ext . u   the fused energy + residual pass (rows a2-a5)
//   loss = sum_{s,k} Pi_{s,k} / (S K)   batch mean (Eq. 2): samples and parts are the batch
//   dloss/dH = phi (.) (f_int(u) - f_ext) / (S K)
// The network itself is out of scope; these are the values its backward consumes.
#include <type_traits>

#include "launch.cuh"

namespace pfem {

constexpr int PT_NT = 256;

// u[s][n][i] = phi[n][i] * H[s][n][i]; VEC: 16-byte vectors (nd and sstride multiples of W)
template <class T, bool VEC>
__global__ void __launch_bounds__(PT_NT)
k_ansatz(int S, int64_t nd, int64_t sstride, const T* __restrict__ H, const T* __restrict__ phi, T* __restrict__ u) {
    constexpr int W = VEC ? 16 / sizeof(T) : 1;
    const int64_t stride = (int64_t)gridDim.x * PT_NT;
    for (int64_t i = ((int64_t)blockIdx.x * PT_NT + threadIdx.x) * W; i < nd; i += stride * W) {
        if constexpr (VEC) {
            using V4 = std::conditional_t<sizeof(T) == 4, float4, double2>;
            const V4 ph = __ldg(reinterpret_cast<const V4*>(phi + i));
            for (int s = 0; s < S; ++s) {
                V4 h = __ldcs(reinterpret_cast<const V4*>(H + (int64_t)s * sstride + i));
                if constexpr (sizeof(T) == 4) {
                    h.x *= ph.x; h.y *= ph.y; h.z *= ph.z; h.w *= ph.w;
                } else {
                    h.x *= ph.x; h.y *= ph.y;
                }
                *reinterpret_cast<V4*>(u + (int64_t)s * sstride + i) = h;
            }
        } else {
            const T ph = phi[i];
            for (int s = 0; s < S; ++s) u[(int64_t)s * sstride + i] = ph * H[(int64_t)s * sstride + i];
        }
    }
}

// g[s][n][i] = phi[n][i] (r[s][n][i] - f[n][i]) * inv  (in place on the residual);
// CTA 0 also forms loss = sum of totals [S][K] in row order, / (S K)
template <class T>
__global__ void __launch_bounds__(PT_NT)
k_pretrain_epilogue(int S, int K, int64_t nd, int64_t sstride, const T* __restrict__ phi, const T* __restrict__ f,
                    T* __restrict__ g, const T* __restrict__ totals, double* __restrict__ loss) {
    const double inv = 1.0 / ((double)S * (double)K);
    const T tinv = (T)inv;
    const int64_t stride = (int64_t)gridDim.x * PT_NT;
    for (int64_t i = (int64_t)blockIdx.x * PT_NT + threadIdx.x; i < nd; i += stride) {
        const T ph = phi ? phi[i] : T(1);
        const T fe = f ? f[i] : T(0);
        for (int s = 0; s < S; ++s) {
            T* gp = g + (int64_t)s * sstride + i;
            *gp = ph * (*gp - fe) * tinv;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && loss) {
        double t = 0.0;
        for (int j = 0; j < S * K; ++j) t += (double)totals[j];
        *loss = t * inv;
    }
}

template <class T>
pfem_status pretrain_epilogue_impl(const pfem_mesh* m, int S, int64_t sstride, const void* H, const void* phi,
                                   void* u, int stage, const void* f_ext, void* grad, const void* totals,
                                   double* loss, cudaStream_t s) {
    const int64_t nd = (int64_t)m->n_nodes * m->dim;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * 148, (nd + PT_NT - 1) / PT_NT));
    if (stage == 0) {
        constexpr int W = 16 / sizeof(T);
        const bool vec = nd % W == 0 && sstride % W == 0 && ((uintptr_t)H | (uintptr_t)phi | (uintptr_t)u) % 16 == 0;
        if (vec) k_ansatz<T, true><<<grid, PT_NT, 0, s>>>(S, nd, sstride, (const T*)H, (const T*)phi, (T*)u);
        else k_ansatz<T, false><<<grid, PT_NT, 0, s>>>(S, nd, sstride, (const T*)H, (const T*)phi, (T*)u);
        PFEM_LAUNCH_CHECK("k_ansatz");
    } else {
        const Plan* P = reinterpret_cast<const Plan*>(m->plan);
        k_pretrain_epilogue<T><<<grid, PT_NT, 0, s>>>(S, P->n_parts, nd, sstride, (const T*)phi, (const T*)f_ext,
                                                      (T*)grad, (const T*)totals, loss);
        PFEM_LAUNCH_CHECK("k_pretrain_epilogue");
    }
    count_launch();
    return PFEM_OK;
}

pfem_status run_pretrain_stage(const pfem_mesh* m, int S, int64_t sstride, const void* H, const void* phi, void* u,
                               int stage, const void* f_ext, void* grad, const void* totals, double* loss,
                               cudaStream_t s) {
    return m->dtype == PFEM_F32
               ? pretrain_epilogue_impl<float>(m, S, sstride, H, phi, u, stage, f_ext, grad, totals, loss, s)
               : pretrain_epilogue_impl<double>(m, S, sstride, H, phi, u, stage, f_ext, grad, totals, loss, s);
}

}  // namespace pfem

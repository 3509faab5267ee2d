// element.cuh — per-element arithmetic of the explicit FE differentiation (device code).
//
//   kinematics  H = sum_{a=1..d} (u_{v_a} - u_{v_0}) (x) grad N_a,  F = I + H
//   linear      eps = sym H, P = sigma = 2 mu eps + lam tr(eps) I, psi = mu eps:eps + lam/2 tr(eps)^2
//               (§4.1: E/(1+nu) = 2 mu, E nu/((1+nu)(1-2nu)) = lam)
//   Neo-Hookean psi = lam/2 (ln J)^2 - mu ln J + mu/2 (I1 - d), P = mu (F - F^-T) + lam ln J F^-T
//               (§4.2; P = F S with S of App. B)
//   forces      f_a = V P grad N_a (App. B P:1086 / P:1096), f_0 = -sum_{a>=1} f_a
//   tangent     dP = mu dH + (mu - lam ln J) F^-T dH^T F^-T + lam (F^-T : dH) F^-T
//
// Cancellation-free evaluation near F = I (exact algebra, so the fp64
// values agree with the plain formulas to rounding):
//   x = J - 1 = tr H + i2(H) + det H (3-D) or tr H + det H (2-D), ln J = log1p(x)
//   psi_NH = lam/2 ln^2 J + mu (|H|^2/2 - i2 - det H + g(x)),  g(x) = x - log1p(x)
//   adj(I+H) = (1 + t + i2) I - (1 + t) H + H^2   (3-D Cayley-Hamilton), (1+t) I - H (2-D)
//   F - F^-T = [det H I + (1+x) H + (1+t) H^T - (H^T)^2] / J  (3-D), [det H I + (1+x) H + H^T] / J (2-D)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pfem {

enum { MODEL_LINEAR = 0, MODEL_NH = 1 };
enum { KIND_LAME = 0, KIND_YP = 1, KIND_YP_PLANE_STRESS = 2 };

template <class T>
struct MatArgs {
    int kind;
    const T* p0;
    const T* p1;
    int64_t s0, s1;
};

template <int D, class T>
struct Geo {
    int v[D + 1];
    T g[D][D];      // g[a][j] = dN_{a+1}/dX_j
    T V;
    T mu, lam;
};

template <class T>
__device__ __forceinline__ T tone() { return T(1); }

// (E, nu) -> (mu, lambda)
template <class T>
__device__ __forceinline__ void lame_of(int kind, T p0, T p1, T& mu, T& lam) {
    if (kind == KIND_LAME) {
        mu = p0;
        lam = p1;
    } else {
        mu = p0 / (T(2) * (T(1) + p1));
        lam = p1 * p0 / ((T(1) + p1) * (T(1) - T(2) * p1));
        if (kind == KIND_YP_PLANE_STRESS) lam = T(2) * mu * lam / (lam + T(2) * mu);
    }
}

template <int D, class T>
__device__ __forceinline__ void load_geo(int e, int E, const int32_t* __restrict__ conn,
                                         const T* __restrict__ grad, const T* __restrict__ vol,
                                         const MatArgs<T>& m, Geo<D, T>& G) {
    if (D == 3) {
        int4 c = __ldg(reinterpret_cast<const int4*>(conn) + e);
        G.v[0] = c.x; G.v[1] = c.y; G.v[2] = c.z; G.v[D == 3 ? 3 : 0] = c.w;
    } else {
#pragma unroll
        for (int a = 0; a <= D; ++a) G.v[a] = __ldg(conn + (int64_t)e * (D + 1) + a);
    }
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int j = 0; j < D; ++j) G.g[a][j] = __ldg(grad + (int64_t)(a * D + j) * E + e);
    G.V = __ldg(vol + e);
    T p0 = __ldg(m.p0 + (int64_t)e * m.s0);
    T p1 = __ldg(m.p1 + (int64_t)e * m.s1);
    lame_of<T>(m.kind, p0, p1, G.mu, G.lam);
}

// gather the d+1 nodal vectors of one sample; masked DOFs read as 0
template <int D, class T, bool MASKED>
__device__ __forceinline__ void gather(const T* __restrict__ f, const uint8_t* __restrict__ mask,
                                       const Geo<D, T>& G, T x[D + 1][D]) {
#pragma unroll
    for (int a = 0; a <= D; ++a) {
        const int64_t base = (int64_t)G.v[a] * D;
        if (D == 2 && sizeof(T) == 8) {
            double2 q = __ldg(reinterpret_cast<const double2*>(f + base));
            x[a][0] = (T)q.x;
            x[a][D - 1] = (T)q.y;
        } else if (D == 2 && sizeof(T) == 4) {
            float2 q = __ldg(reinterpret_cast<const float2*>(f + base));
            x[a][0] = (T)q.x;
            x[a][D - 1] = (T)q.y;
        } else {
#pragma unroll
            for (int i = 0; i < D; ++i) x[a][i] = __ldg(f + base + i);
        }
        if (MASKED) {
#pragma unroll
            for (int i = 0; i < D; ++i)
                if (__ldg(mask + base + i)) x[a][i] = T(0);
        }
    }
}

// H = sum_{a=1..d} (x_a - x_0) (x) g_{a-1}
template <int D, class T>
__device__ __forceinline__ void grad_of(const Geo<D, T>& G, const T x[D + 1][D], T H[D][D]) {
    T dx[D][D];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) dx[a][i] = x[a + 1][i] - x[0][i];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            T s = dx[0][i] * G.g[0][j];
#pragma unroll
            for (int a = 1; a < D; ++a) s = fma(dx[a][i], G.g[a][j], s);
            H[i][j] = s;
        }
}

// g(x) = x - log1p(x) without cancellation: with z = x/(2+x), log1p(x) = 2 atanh z, so
// g = x^2/(2+x) - 2 (z^3/3 + z^5/5 + ...)   (|x| < 1/2), direct form otherwise.
template <class T>
__device__ __forceinline__ T g_of(T x) {
    if (fabs(x) < T(0.5)) {
        T r = T(1) / (T(2) + x);
        T z = x * r;
        T z2 = z * z;
        T s;
        if (sizeof(T) == 4) {
            s = T(1.0 / 11);
            s = fma(s, z2, T(1.0 / 9));
            s = fma(s, z2, T(1.0 / 7));
            s = fma(s, z2, T(1.0 / 5));
            s = fma(s, z2, T(1.0 / 3));
        } else {
            s = T(1.0 / 27);
#pragma unroll
            for (int k = 25; k >= 3; k -= 2) s = fma(s, z2, T(1.0) / T(k));
        }
        return x * x * r - T(2) * z * z2 * s;
    }
    return x - log1p(x);
}

// Neo-Hookean state from H: x = J-1, lnJ, 1/J, F^-T (A), and optionally psi
template <int D, class T>
struct NhState {
    T x, lnJ, invJ, t, i2, detH;
    T A[D][D];   // F^-T = cof(F) / J
};

template <int D, class T>
__device__ __forceinline__ void nh_state(const T H[D][D], NhState<D, T>& S, T H2[D][D]) {
    if (D == 2) {
        S.t = H[0][0] + H[1][1];
        S.detH = H[0][0] * H[1][1] - H[0][1] * H[1][0];
        S.i2 = T(0);
        S.x = S.t + S.detH;
    } else {
        S.t = H[0][0] + H[1][1] + H[D - 1][D - 1];
        // H2 = H H
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                T s = H[i][0] * H[0][j];
#pragma unroll
                for (int k = 1; k < D; ++k) s = fma(H[i][k], H[k][j], s);
                H2[i][j] = s;
            }
        T trH2 = H2[0][0] + H2[1][1] + H2[D - 1][D - 1];
        S.i2 = T(0.5) * (S.t * S.t - trH2);
        // det H by cofactor expansion on row 0
        S.detH = H[0][0] * (H[1][1] * H[D - 1][D - 1] - H[1][D - 1] * H[D - 1][1]) -
                 H[0][1] * (H[1][0] * H[D - 1][D - 1] - H[1][D - 1] * H[D - 1][0]) +
                 H[0][D - 1] * (H[1][0] * H[D - 1][1] - H[1][1] * H[D - 1][0]);
        S.x = S.t + S.i2 + S.detH;
    }
    S.lnJ = log1p(S.x);
    S.invJ = T(1) / (T(1) + S.x);
    // cof(F) = adj(F)^T
    if (D == 2) {
        // adj = (1+t) I - H  ->  cof = (1+t) I - H^T
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j)
                S.A[i][j] = ((i == j ? T(1) + S.t : T(0)) - H[j][i]) * S.invJ;
    } else {
        // adj = (1+t+i2) I - (1+t) H + H^2  ->  cof = (1+t+i2) I - (1+t) H^T + (H^2)^T
        const T c0 = T(1) + S.t + S.i2, c1 = T(1) + S.t;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j)
                S.A[i][j] = ((i == j ? c0 : T(0)) - c1 * H[j][i] + H2[j][i]) * S.invJ;
    }
}

// first Piola stress and (optionally) the energy density
template <int D, int MODEL, class T, bool WANT_PSI>
__device__ __forceinline__ void stress(const Geo<D, T>& G, const T H[D][D], T P[D][D], T& psi,
                                       bool& bad) {
    if (MODEL == MODEL_LINEAR) {
        T tr = H[0][0];
#pragma unroll
        for (int i = 1; i < D; ++i) tr += H[i][i];
        T ee = T(0);
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                T eps = T(0.5) * (H[i][j] + H[j][i]);
                P[i][j] = T(2) * G.mu * eps + (i == j ? G.lam * tr : T(0));
                if (WANT_PSI) ee = fma(eps, eps, ee);
            }
        if (WANT_PSI) psi = G.mu * ee + T(0.5) * G.lam * tr * tr;
        bad = false;
    } else {
        NhState<D, T> S;
        T H2[D][D];
        nh_state<D, T>(H, S, H2);
        bad = !(S.x > T(-1));
        // F - F^-T
        T Dm[D][D];
        if (D == 2) {
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j)
                    Dm[i][j] = ((i == j ? S.detH : T(0)) + (T(1) + S.x) * H[i][j] + H[j][i]) * S.invJ;
        } else {
            const T c1 = T(1) + S.t;
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j)
                    Dm[i][j] = ((i == j ? S.detH : T(0)) + (T(1) + S.x) * H[i][j] + c1 * H[j][i] - H2[j][i]) *
                               S.invJ;
        }
        const T ll = G.lam * S.lnJ;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) P[i][j] = G.mu * Dm[i][j] + ll * S.A[i][j];
        if (WANT_PSI) {
            T hh = T(0);
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) hh = fma(H[i][j], H[i][j], hh);
            psi = T(0.5) * G.lam * S.lnJ * S.lnJ + G.mu * (T(0.5) * hh - S.i2 - S.detH + g_of<T>(S.x));
        }
    }
}

// tangent stress increment dP(dH) at state H (NH) or for the linear law
template <int D, int MODEL, class T>
__device__ __forceinline__ void dstress(const Geo<D, T>& G, const NhState<D, T>& S, const T dH[D][D],
                                        T dP[D][D]) {
    if (MODEL == MODEL_LINEAR) {
        T tr = dH[0][0];
#pragma unroll
        for (int i = 1; i < D; ++i) tr += dH[i][i];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j)
                dP[i][j] = G.mu * (dH[i][j] + dH[j][i]) + (i == j ? G.lam * tr : T(0));
    } else {
        // M1 = A dH^T ; M2 = M1 A ; tr(F^-1 dH) = A : dH
        T M1[D][D];
        T tr = T(0);
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                T s = S.A[i][0] * dH[j][0];
#pragma unroll
                for (int k = 1; k < D; ++k) s = fma(S.A[i][k], dH[j][k], s);
                M1[i][j] = s;
                tr = fma(S.A[i][j], dH[i][j], tr);
            }
        const T c = G.mu - G.lam * S.lnJ;
        const T lt = G.lam * tr;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                T s = M1[i][0] * S.A[0][j];
#pragma unroll
                for (int k = 1; k < D; ++k) s = fma(M1[i][k], S.A[k][j], s);
                dP[i][j] = G.mu * dH[i][j] + c * s + lt * S.A[i][j];
            }
    }
}

// nodal forces f[a][i], a = 0..d, from P (already including nothing of V)
template <int D, class T>
__device__ __forceinline__ void forces(const Geo<D, T>& G, const T P[D][D], T f[D + 1][D]) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
        T s0 = T(0);
#pragma unroll
        for (int a = 0; a < D; ++a) {
            T s = P[i][0] * G.g[a][0];
#pragma unroll
            for (int j = 1; j < D; ++j) s = fma(P[i][j], G.g[a][j], s);
            s *= G.V;
            f[a + 1][i] = s;
            s0 -= s;
        }
        f[0][i] = s0;
    }
}

}  // namespace pfem

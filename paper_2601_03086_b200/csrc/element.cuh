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
// Evaluation near F = I (exact algebra, so fp64 agrees with the plain
// formulas to rounding; fp32 avoids the catastrophic cancellation of the energy):
//   x = J - 1 = tr H + i2(H) + det H (3-D) or tr H + det H (2-D)
//   ln J = log1p(x) = 2 atanh(z), z = x / (2 + x);   g(x) = x - log1p(x) = x^2/(2+x) - 2 (z^3/3 + z^5/5 + ..)
//   psi_NH = lam/2 ln^2 J + mu (|H|^2/2 - i2 - det H + g(x))
//   P = mu F + (lam ln J - mu) cof(F) / J        (F^-T = cof(F) / J)
// One-point quadrature: V_e is folded into (mu, lambda) at load time.
//
// The arithmetic is written once for a value type V: double, float, or F2 (two samples
// that share the element's geometry in one sm_100a FFMA2 / FADD2 / FMUL2 register pair;
// the geometry stays a scalar operand, which FFMA2 broadcasts for free).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pfem {

enum { MODEL_LINEAR = 0, MODEL_NH = 1 };
enum { KIND_LAME = 0, KIND_YP = 1, KIND_YP_PLANE_STRESS = 2 };

// ------------------------------------------------------------------ F2: 2 x fp32 lanes
struct F2 {
    float2 v;
    __device__ __forceinline__ F2() {}
    __device__ __forceinline__ explicit F2(float s) : v(make_float2(s, s)) {}
    __device__ __forceinline__ F2(float a, float b) : v(make_float2(a, b)) {}
};
__device__ __forceinline__ F2 operator+(F2 a, F2 b) { F2 r; r.v = __fadd2_rn(a.v, b.v); return r; }
__device__ __forceinline__ F2 operator-(F2 a, F2 b) { F2 r; r.v = __fadd2_rn(a.v, make_float2(-b.v.x, -b.v.y)); return r; }
__device__ __forceinline__ F2 operator-(F2 a) { return F2(-a.v.x, -a.v.y); }
__device__ __forceinline__ F2 operator*(F2 a, F2 b) { F2 r; r.v = __fmul2_rn(a.v, b.v); return r; }
__device__ __forceinline__ F2 operator+(F2 a, float b) { return a + F2(b); }
__device__ __forceinline__ F2 operator+(float a, F2 b) { return F2(a) + b; }
__device__ __forceinline__ F2 operator-(F2 a, float b) { return a - F2(b); }
__device__ __forceinline__ F2 operator-(float a, F2 b) { return F2(a) - b; }
__device__ __forceinline__ F2 operator*(F2 a, float b) { return a * F2(b); }
__device__ __forceinline__ F2 operator*(float a, F2 b) { return F2(a) * b; }
__device__ __forceinline__ F2& operator+=(F2& a, F2 b) { a = a + b; return a; }
__device__ __forceinline__ F2 fma(F2 a, F2 b, F2 c) { F2 r; r.v = __ffma2_rn(a.v, b.v, c.v); return r; }
__device__ __forceinline__ F2 fma(F2 a, float b, F2 c) { return fma(a, F2(b), c); }
__device__ __forceinline__ F2 fma(float a, F2 b, F2 c) { return fma(F2(a), b, c); }
using ::fma;   // keep the float / double overloads visible next to the F2 ones

// ------------------------------------------------------------------ F4: 4 x fp32 lanes (two F2)
// Four samples of one element in lockstep: every operation is two independent FFMA2 / FADD2 /
// FMUL2, which doubles the instruction-level parallelism of the element arithmetic, and the
// staged fields / force buffer move 16 bytes per shared-memory access.
struct __align__(16) F4 {
    F2 a, b;
    __device__ __forceinline__ F4() {}
    __device__ __forceinline__ explicit F4(float s) : a(s), b(s) {}
    __device__ __forceinline__ F4(F2 x, F2 y) : a(x), b(y) {}
};
__device__ __forceinline__ F4 operator+(F4 x, F4 y) { return F4(x.a + y.a, x.b + y.b); }
__device__ __forceinline__ F4 operator-(F4 x, F4 y) { return F4(x.a - y.a, x.b - y.b); }
__device__ __forceinline__ F4 operator-(F4 x) { return F4(-x.a, -x.b); }
__device__ __forceinline__ F4 operator*(F4 x, F4 y) { return F4(x.a * y.a, x.b * y.b); }
__device__ __forceinline__ F4 operator+(F4 x, float y) { return F4(x.a + y, x.b + y); }
__device__ __forceinline__ F4 operator+(float x, F4 y) { return F4(x + y.a, x + y.b); }
__device__ __forceinline__ F4 operator-(F4 x, float y) { return F4(x.a - y, x.b - y); }
__device__ __forceinline__ F4 operator-(float x, F4 y) { return F4(x - y.a, x - y.b); }
__device__ __forceinline__ F4 operator*(F4 x, float y) { return F4(x.a * y, x.b * y); }
__device__ __forceinline__ F4 operator*(float x, F4 y) { return F4(x * y.a, x * y.b); }
__device__ __forceinline__ F4& operator+=(F4& x, F4 y) { x = x + y; return x; }
__device__ __forceinline__ F4 fma(F4 x, F4 y, F4 z) { return F4(fma(x.a, y.a, z.a), fma(x.b, y.b, z.b)); }
__device__ __forceinline__ F4 fma(F4 x, float y, F4 z) { return F4(fma(x.a, y, z.a), fma(x.b, y, z.b)); }
__device__ __forceinline__ F4 fma(float x, F4 y, F4 z) { return F4(fma(x, y.a, z.a), fma(x, y.b, z.b)); }

template <class V> struct VTraits;
template <> struct VTraits<float> { using S = float; static constexpr int L = 1; };
template <> struct VTraits<double> { using S = double; static constexpr int L = 1; };
template <> struct VTraits<F2> { using S = float; static constexpr int L = 2; };
template <> struct VTraits<F4> { using S = float; static constexpr int L = 4; };

__device__ __forceinline__ float lane(float x, int) { return x; }
__device__ __forceinline__ double lane(double x, int) { return x; }
__device__ __forceinline__ float lane(F2 x, int k) { return k ? x.v.y : x.v.x; }
__device__ __forceinline__ float lane(F4 x, int k) { return k < 2 ? lane(x.a, k) : lane(x.b, k - 2); }
__device__ __forceinline__ void set_lane(float& x, int, float s) { x = s; }
__device__ __forceinline__ void set_lane(double& x, int, double s) { x = s; }
__device__ __forceinline__ void set_lane(F2& x, int k, float s) { if (k) x.v.y = s; else x.v.x = s; }
__device__ __forceinline__ void set_lane(F4& x, int k, float s) { if (k < 2) set_lane(x.a, k, s); else set_lane(x.b, k - 2, s); }

// reciprocal: fp32 MUFU.RCP + one Newton step (~0.5 ulp); fp64 IEEE division
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ double vrcp(double x) { return 1.0 / x; }
__device__ __forceinline__ float vrcp(float x) {
    float r = rcp_approx(x);
    return fmaf(r, fmaf(-x, r, 1.0f), r);
}
__device__ __forceinline__ F2 vrcp(F2 x) {
    F2 r(rcp_approx(x.v.x), rcp_approx(x.v.y));
    return fma(r, fma(-x, r, F2(1.0f)), r);
}
__device__ __forceinline__ F4 vrcp(F4 x) { return F4(vrcp(x.a), vrcp(x.b)); }

// ln J = log1p(x) and g(x) = x - log1p(x) >= 0 together, cancellation-free.
// |x| < 1/2: z = x/(2+x) (|z| < 1/3), log1p = 2 z (1 + z^2 s(z^2)), g = x^2/(2+x) - 2 z^3 s(z^2),
// s = 1/3 + z^2/5 + ...; else the library log1p.
__device__ __forceinline__ void log1p_g(double x, double& l, double& g) {
    if (fabs(x) < 0.5) {
        const double r = 1.0 / (2.0 + x), z = x * r, z2 = z * z;
        double s = 1.0 / 41;
#pragma unroll
        for (int k = 39; k >= 3; k -= 2) s = fma(s, z2, 1.0 / k);
        const double zs = z * z2 * s;
        l = 2.0 * (z + zs);
        g = fma(x * x, r, -2.0 * zs);
    } else {
        l = log1p(x);
        g = x - l;
    }
}
template <class V>
__device__ __forceinline__ void log1p_g(V x, V& l, V& g) {   // float / F2
    bool small = true;
#pragma unroll
    for (int k = 0; k < VTraits<V>::L; ++k) small = small && fabsf(lane(x, k)) < 0.5f;
    if (small) {
        const V r = vrcp(x + 2.0f), z = x * r, z2 = z * z;
        V s = fma(z2, 1.0f / 15, V(1.0f / 13));
        s = fma(s, z2, V(1.0f / 11));
        s = fma(s, z2, V(1.0f / 9));
        s = fma(s, z2, V(1.0f / 7));
        s = fma(s, z2, V(1.0f / 5));
        s = fma(s, z2, V(1.0f / 3));
        const V zs = z * z2 * s;
        l = 2.0f * (z + zs);
        g = fma(x * x, r, -2.0f * zs);
    } else {
#pragma unroll
        for (int k = 0; k < VTraits<V>::L; ++k) {
            const float xl = lane(x, k), ll = log1pf(xl);
            set_lane(l, k, ll);
            set_lane(g, k, xl - ll);
        }
    }
}

// P1 geometry from the d+1 vertex coordinates, fp64 (App. B):
// J = [X_1-X_0 | .. | X_d-X_0] (columns), inv = J^{-1} (row a = grad N_{a+1}), returns det J.
// The one formula of both the prepared geometry (k_geometry) and the on-the-fly option.
template <int D>
__device__ __forceinline__ double geometry_of(const double (&X)[D + 1][D], double (&inv)[D][D]) {
    double J[D][D];
#pragma unroll
    for (int a = 1; a <= D; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) J[i][a - 1] = X[a][i] - X[0][i];
    double det;
    if constexpr (D == 2) {
        det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        const double r = 1.0 / det;
        inv[0][0] = J[1][1] * r;
        inv[0][1] = -J[0][1] * r;
        inv[1][0] = -J[1][0] * r;
        inv[1][1] = J[0][0] * r;
    } else {
        // cofactors of J: C_ij; inverse = C^T / det
        const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
        const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
        const double r = 1.0 / det;
        inv[0][0] = c00 * r;
        inv[1][0] = c01 * r;
        inv[2][0] = c02 * r;
        inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * r;
        inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * r;
        inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * r;
        inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * r;
        inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * r;
        inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * r;
    }
    return det;
}

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
    T mu, lam;      // V_e * mu, V_e * lambda after load_geo
};

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

// (E, nu) with a uniform nu: both moduli are E times a constant, (mu, lambda) = E (mu_1, lambda_1)
// with (mu_1, lambda_1) = lame(1, nu) formed once per thread, so the per-element work is two
// multiplies instead of two divisions (1 ulp from the quotient form)
template <class T>
struct LameScale {
    T mu1, lam1;
    bool on;
};

template <class T>
__device__ __forceinline__ LameScale<T> lame_scale(const MatArgs<T>& m) {
    LameScale<T> L;
    L.on = m.kind != KIND_LAME && m.s1 == 0;
    L.mu1 = L.lam1 = T(0);
    if (L.on) lame_of<T>(m.kind, T(1), __ldg(m.p1), L.mu1, L.lam1);
    return L;
}

template <class T>
__device__ __forceinline__ void lame_elem(const MatArgs<T>& m, const LameScale<T>& L, T p0, T p1, T& mu, T& lam) {
    if (L.on) {
        mu = p0 * L.mu1;
        lam = p0 * L.lam1;
    } else {
        lame_of<T>(m.kind, p0, p1, mu, lam);
    }
}

template <int D, class T>
__device__ __forceinline__ void load_geo(int e, int E, const int32_t* __restrict__ conn,
                                         const T* __restrict__ grad, const T* __restrict__ vol,
                                         const MatArgs<T>& m, Geo<D, T>& G) {
    if constexpr (D == 3) {
        int4 c = __ldg(reinterpret_cast<const int4*>(conn) + e);
        G.v[0] = c.x; G.v[1] = c.y; G.v[2] = c.z; G.v[3] = c.w;
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
    // one-point quadrature: fold V_e into the moduli, so psi -> W_e = V_e psi and
    // P -> V_e P (forces f_a = (V_e P) grad N_a need no further scaling)
    G.mu *= G.V;
    G.lam *= G.V;
}

// gather the d+1 nodal vectors of L consecutive samples (stride sstride); masked DOFs -> 0
template <int D, class T, class V, bool MASKED>
__device__ __forceinline__ void gather(const T* __restrict__ f, int64_t sstride, const uint8_t* __restrict__ mask,
                                       const Geo<D, T>& G, V x[D + 1][D]) {
#pragma unroll
    for (int a = 0; a <= D; ++a) {
        const int base = G.v[a] * D;
#pragma unroll
        for (int k = 0; k < VTraits<V>::L; ++k) {
            const T* fk = f + k * sstride + base;
            if constexpr (D == 2 && sizeof(T) == 8) {
                double2 q = __ldg(reinterpret_cast<const double2*>(fk));
                set_lane(x[a][0], k, q.x);
                set_lane(x[a][D - 1], k, q.y);
            } else if constexpr (D == 2 && sizeof(T) == 4) {
                float2 q = __ldg(reinterpret_cast<const float2*>(fk));
                set_lane(x[a][0], k, q.x);
                set_lane(x[a][D - 1], k, q.y);
            } else {
#pragma unroll
                for (int i = 0; i < D; ++i) set_lane(x[a][i], k, __ldg(fk + i));
            }
        }
        if (MASKED) {
#pragma unroll
            for (int i = 0; i < D; ++i)
                if (__ldg(mask + base + i)) x[a][i] = V(T(0));
        }
    }
}

// H = sum_{a=1..d} (x_a - x_0) (x) g_{a-1}
template <int D, class T, class V>
__device__ __forceinline__ void grad_of(const Geo<D, T>& G, const V x[D + 1][D], V H[D][D]) {
    V dx[D][D];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) dx[a][i] = x[a + 1][i] - x[0][i];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            V s = dx[0][i] * G.g[0][j];
#pragma unroll
            for (int a = 1; a < D; ++a) s = fma(dx[a][i], G.g[a][j], s);
            H[i][j] = s;
        }
}

template <int D, class V>
__device__ __forceinline__ void cofactor(const V F[D][D], V cof[D][D]) {
    if constexpr (D == 2) {
        cof[0][0] = F[1][1];
        cof[0][1] = -F[1][0];
        cof[1][0] = -F[0][1];
        cof[1][1] = F[0][0];
    } else {
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const int i1 = (i + 1) % D, i2 = (i + 2) % D, j1 = (j + 1) % D, j2 = (j + 2) % D;
                cof[i][j] = fma(F[i1][j1], F[i2][j2], -(F[i1][j2] * F[i2][j1]));
            }
    }
}

// count of lanes with !(x > -1) (J <= 0 or NaN)
template <class V>
__device__ __forceinline__ int n_bad(V x) {
    int n = 0;
#pragma unroll
    for (int k = 0; k < VTraits<V>::L; ++k) n += !(lane(x, k) > -1.0f) ? 1 : 0;
    return n;
}

// Neo-Hookean linearisation state from H (tangent): ln J, A = F^-T = cof(F) / J
template <int D, class V>
struct NhState {
    V x, lnJ;
    V A[D][D];
};

template <int D, class V>
__device__ __forceinline__ void nh_state(const V H[D][D], NhState<D, V>& S) {
    V F[D][D], cof[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) F[i][j] = (i == j) ? H[i][j] + 1.0f : H[i][j];
    cofactor<D, V>(F, cof);
    V J = F[0][0] * cof[0][0];
#pragma unroll
    for (int j = 1; j < D; ++j) J = fma(F[0][j], cof[0][j], J);
    S.x = J - 1.0f;
    V g;
    log1p_g(S.x, S.lnJ, g);
    const V invJ = vrcp(J);
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) S.A[i][j] = cof[i][j] * invJ;
}

// first Piola stress (times V_e) and, if WANT_PSI, the element energy W_e = V_e psi
template <int D, int MODEL, class T, class V, bool WANT_PSI>
__device__ __forceinline__ void stress(const Geo<D, T>& G, const V H[D][D], V P[D][D], V& psi, int& bad) {
    if constexpr (MODEL == MODEL_LINEAR) {
        V tr = H[0][0];
#pragma unroll
        for (int i = 1; i < D; ++i) tr = tr + H[i][i];
        const V lt = G.lam * tr;
        V ee = V(T(0));
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                if (i == j) {
                    P[i][i] = fma(H[i][i], T(2) * G.mu, lt);
                    if (WANT_PSI) ee = fma(H[i][i], H[i][i], ee);
                } else if (j > i) {
                    const V s = H[i][j] + H[j][i];          // 2 eps_ij
                    P[i][j] = s * G.mu;
                    P[j][i] = P[i][j];
                    if (WANT_PSI) ee = fma(s, s * T(0.5), ee);   // eps_ij^2 + eps_ji^2
                }
            }
        if (WANT_PSI) psi = fma(ee, G.mu, (G.lam * T(0.5)) * (tr * tr));
        bad = 0;
    } else {
        V t = H[0][0];
#pragma unroll
        for (int i = 1; i < D; ++i) t = t + H[i][i];
        V detH, i2 = V(T(0));
        if constexpr (D == 2) {
            detH = fma(H[0][0], H[1][1], -(H[0][1] * H[1][0]));
        } else {
            V trH2 = H[0][0] * H[0][0];
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j)
                    if (i || j) trH2 = fma(H[i][j], H[j][i], trH2);
            i2 = fma(t, t, -trH2) * T(0.5);
            const V m0 = fma(H[1][1], H[2][2], -(H[1][2] * H[2][1]));
            const V m1 = fma(H[1][0], H[2][2], -(H[1][2] * H[2][0]));
            const V m2 = fma(H[1][0], H[2][1], -(H[1][1] * H[2][0]));
            detH = fma(H[0][0], m0, fma(-H[0][1], m1, H[0][2] * m2));
        }
        const V x = t + i2 + detH;
        bad = n_bad(x);
        V lnJ, g;
        log1p_g(x, lnJ, g);
        const V invJ = vrcp(x + T(1));
        V F[D][D], cof[D][D];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) F[i][j] = (i == j) ? H[i][j] + T(1) : H[i][j];
        cofactor<D, V>(F, cof);
        const V c = fma(lnJ, G.lam, V(-G.mu)) * invJ;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) P[i][j] = fma(c, cof[i][j], F[i][j] * G.mu);
        if (WANT_PSI) {
            V hh = H[0][0] * H[0][0];
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j)
                    if (i || j) hh = fma(H[i][j], H[i][j], hh);
            const V inner = fma(hh, T(0.5), g - i2 - detH);
            psi = fma((G.lam * T(0.5)) * lnJ, lnJ, inner * G.mu);
        }
    }
}

// tangent stress increment dP(dH) at state S (NH) or for the linear law (times V_e)
template <int D, int MODEL, class T, class V>
__device__ __forceinline__ void dstress(const Geo<D, T>& G, const NhState<D, V>& S, const V dH[D][D], V dP[D][D]) {
    if constexpr (MODEL == MODEL_LINEAR) {
        V tr = dH[0][0];
#pragma unroll
        for (int i = 1; i < D; ++i) tr = tr + dH[i][i];
        const V lt = G.lam * tr;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                if (i == j) dP[i][i] = fma(dH[i][i], T(2) * G.mu, lt);
                else if (j > i) {
                    dP[i][j] = (dH[i][j] + dH[j][i]) * G.mu;
                    dP[j][i] = dP[i][j];
                }
            }
    } else {
        // M1 = A dH^T ; M2 = M1 A ; tr(F^-1 dH) = A : dH
        V M1[D][D];
        V tr = S.A[0][0] * dH[0][0];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                V s = S.A[i][0] * dH[j][0];
#pragma unroll
                for (int k = 1; k < D; ++k) s = fma(S.A[i][k], dH[j][k], s);
                M1[i][j] = s;
                if (i || j) tr = fma(S.A[i][j], dH[i][j], tr);
            }
        const V cc = fma(S.lnJ, -G.lam, V(G.mu));
        const V lt = tr * G.lam;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                V s = M1[i][0] * S.A[0][j];
#pragma unroll
                for (int k = 1; k < D; ++k) s = fma(M1[i][k], S.A[k][j], s);
                dP[i][j] = fma(cc, s, fma(lt, S.A[i][j], dH[i][j] * G.mu));
            }
    }
}

// nodal forces f[a][i] = (V P) grad N_a, a = 0..d (V already folded into P via the moduli)
template <int D, class T, class V>
__device__ __forceinline__ void forces(const Geo<D, T>& G, const V P[D][D], V f[D + 1][D]) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
        V s0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            V s = P[i][0] * G.g[a][0];
#pragma unroll
            for (int j = 1; j < D; ++j) s = fma(P[i][j], G.g[a][j], s);
            f[a + 1][i] = s;
            s0 = (a == 0) ? -s : s0 - s;
        }
        f[0][i] = s0;
    }
}

}  // namespace pfem

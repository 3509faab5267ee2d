/*
 * pfem_oracle.c — plain, slow, obviously-correct CPU reference ("oracle") for the
 * PFEM explicit-FE hot path (arXiv 2601.03086).  TEST INFRASTRUCTURE ONLY: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  It shares no code, header, table or helper with
 * the CUDA path (paper_2601_03086_b200/csrc); it follows the paper's textbook
 * formulations, not the GPU's:
 *
 *   geometry       P1 shape functions, grad N_a = rows of J^{-1}      (App. B)
 *   linear energy  Psi = 1/2 sigma:eps, sigma = E/(1+nu) eps + E nu/((1+nu)(1-2nu)) tr(eps) I   (§4.1 eq.)
 *   Neo-Hookean    Psi = 1/2 lam (ln J)^2 - mu ln J + 1/2 mu (I1 - d)  (§4.2 eq.; reading R2: "-2" -> "-d")
 *   Lame           lam = nu E/((1+nu)(1-2nu)), mu = E/(2(1+nu))        (§4.2)
 *   residual       f_int_iI = int dN_I/dX_l F_ik S_kl dV0 (total Lagrangian, App. B);
 *                  linear: f = int B^T sigma dV (virtual power)
 *   tangent        K = int G0^T S G0 + B0^T C^SE B0 dV0                 (App. B); linear: B^T D B
 *   CG             K U = F, stop on ||K U - F|| / ||F|| < tol            (App. B), warm start U0
 *   Jacobi PCG     M = diag of the textbook element tangents, textbook PCG (§5.5; reading R27)
 *   heat           W = 1/2 k |grad T|^2 V, flux = dW/dT                  (Eq. poisson, energy form P:249-284)
 *   (the Newton iteration and the pretraining loss are compositions of these in oracle.py)
 *
 * Everything in float64, plain loops, IEEE RN, built with -O2 -ffp-contract=off.
 * Element-local work may run in an OpenMP parallel loop writing per-element
 * buffers; every assembly (sum into nodes) is a single sequential loop in
 * ascending (element, local node) order.
 *
 * Parity pins: see tests/test_oracle_*.py (closed forms, invariants, finite
 * differences, brute force).  Functions without a pin say "parity unpinned" —
 * currently none.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_ARG (-1)
#define OR_ERR_DEGENERATE (-2)
#define OR_ERR_INVERTED (-3)
#define OR_ERR_NOT_CONVERGED (-4)
#define OR_ERR_BREAKDOWN (-5)
#define OR_ERR_CAPACITY (-6)

#define OR_LINEAR 0
#define OR_NEOHOOKEAN 1

static int64_t g_err_index = -1;
int64_t oracle_last_error_index(void) { return g_err_index; }

/* ------------------------------------------------------------------ */
/* small dense helpers (plain textbook formulas)                       */
/* ------------------------------------------------------------------ */
static double det2(const double A[2][2]) { return A[0][0] * A[1][1] - A[0][1] * A[1][0]; }

static double det3(const double A[3][3]) {
    return A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1])
         - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0])
         + A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
}

/* inverse by adjugate / determinant; returns det */
static double inv_dd(int d, const double A[3][3], double Ai[3][3]) {
    if (d == 2) {
        double a[2][2] = {{A[0][0], A[0][1]}, {A[1][0], A[1][1]}};
        double det = det2(a);
        Ai[0][0] = A[1][1] / det;  Ai[0][1] = -A[0][1] / det;
        Ai[1][0] = -A[1][0] / det; Ai[1][1] = A[0][0] / det;
        return det;
    }
    double det = det3(A);
    Ai[0][0] = (A[1][1] * A[2][2] - A[1][2] * A[2][1]) / det;
    Ai[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) / det;
    Ai[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / det;
    Ai[1][0] = (A[1][2] * A[2][0] - A[1][0] * A[2][2]) / det;
    Ai[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / det;
    Ai[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) / det;
    Ai[2][0] = (A[1][0] * A[2][1] - A[1][1] * A[2][0]) / det;
    Ai[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) / det;
    Ai[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / det;
    return det;
}

/* ------------------------------------------------------------------ */
/* Material: Lame parameters from (E, nu)  — P:727-732                 */
/* kind 0: (mu, lambda) given; 1: (E, nu) plane strain / 3-D;          */
/* 2: (E, nu) plane stress lambda* = 2 mu lam / (lam + 2 mu) (reading R1) */
/* ------------------------------------------------------------------ */
int oracle_lame(int kind, int64_t n, const double* p0, int64_t s0, const double* p1, int64_t s1,
                double* mu, double* lam) {
    for (int64_t e = 0; e < n; ++e) {
        double a = p0[e * s0], b = p1[e * s1];
        if (kind == 0) {
            mu[e] = a;
            lam[e] = b;
        } else {
            double E = a, nu = b;
            double m = E / (2.0 * (1.0 + nu));
            double l = nu * E / ((1.0 + nu) * (1.0 - 2.0 * nu));
            if (kind == 2) l = 2.0 * m * l / (l + 2.0 * m);
            else if (kind != 1) return OR_ERR_ARG;
            mu[e] = m;
            lam[e] = l;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Geometry: J_e = [X_1-X_0 | ... | X_d-X_0] (columns), grad N_a = row  */
/* (a-1) of J^{-1} (a = 1..d), grad N_0 = -sum_a grad N_a,             */
/* V_e = |det J| / d!   (P1 simplex, one-point rule exact) */
/* grad out: [E][d][d] with grad[e][a-1][j] = dN_a/dX_j                */
/* ------------------------------------------------------------------ */
int oracle_geometry(int dim, int64_t n_nodes, int64_t n_elems, const double* coords,
                    const int32_t* conn, double* grad, double* vol, int32_t* sign) {
    if (dim != 2 && dim != 3) return OR_ERR_ARG;
    const int nv = dim + 1;
    for (int64_t e = 0; e < n_elems; ++e)
        for (int a = 0; a < nv; ++a) {
            int32_t v = conn[e * nv + a];
            if (v < 0 || v >= n_nodes) { g_err_index = e; return OR_ERR_ARG; }
        }
    int status = OR_OK;
    int64_t bad = -1;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n_elems; ++e) {
        double J[3][3] = {{0}}, Ji[3][3];
        const int32_t* c = conn + e * nv;
        double edge_prod = 1.0;
        for (int a = 1; a <= dim; ++a) {
            double len2 = 0.0;
            for (int i = 0; i < dim; ++i) {
                J[i][a - 1] = coords[(int64_t)c[a] * dim + i] - coords[(int64_t)c[0] * dim + i];
                len2 += J[i][a - 1] * J[i][a - 1];
            }
            edge_prod *= sqrt(len2);
        }
        double det = inv_dd(dim, J, Ji);
        if (!(fabs(det) > 64.0 * 2.220446049250313e-16 * edge_prod)) {
#pragma omp critical
            { if (bad < 0 || e < bad) bad = e; }
            continue;
        }
        for (int a = 0; a < dim; ++a)
            for (int j = 0; j < dim; ++j) grad[(e * dim + a) * dim + j] = Ji[a][j];
        vol[e] = fabs(det) / (dim == 2 ? 2.0 : 6.0);
        if (sign) sign[e] = det > 0 ? 1 : -1;
    }
    if (bad >= 0) { g_err_index = bad; status = OR_ERR_DEGENERATE; }
    return status;
}

/* all d+1 gradients of element e: g[a][j], a = 0..d */
static void elem_grads(int dim, const double* grad, int64_t e, double g[4][3]) {
    for (int j = 0; j < dim; ++j) {
        double s = 0.0;
        for (int a = 1; a <= dim; ++a) {
            g[a][j] = grad[(e * dim + (a - 1)) * dim + j];
            s += g[a][j];
        }
        g[0][j] = -s;
    }
}

/* ------------------------------------------------------------------ */
/* node -> (element, slot) CSR: entries of node n are all (e, a) with   */
/* conn[e][a] == n in ascending (e, a), stored as e*(d+1)+a (reading R12) */
/* ------------------------------------------------------------------ */
int oracle_csr(int dim, int64_t n_nodes, int64_t n_elems, const int32_t* conn,
               int32_t* ptr, int32_t* ent) {
    const int nv = dim + 1;
    int64_t* fill = (int64_t*)calloc((size_t)n_nodes, sizeof(int64_t));
    if (!fill) return OR_ERR_CAPACITY;
    for (int64_t n = 0; n <= n_nodes; ++n) ptr[n] = 0;
    for (int64_t k = 0; k < n_elems * nv; ++k) ptr[conn[k] + 1] += 1;
    for (int64_t n = 0; n < n_nodes; ++n) ptr[n + 1] += ptr[n];
    for (int64_t e = 0; e < n_elems; ++e)          /* ascending (e, a): rows come out sorted */
        for (int a = 0; a < nv; ++a) {
            int32_t n = conn[e * nv + a];
            ent[ptr[n] + fill[n]] = (int32_t)(e * nv + a);
            fill[n] += 1;
        }
    free(fill);
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Greedy first-fit colouring in ascending element id (reading R12):   */
/* colour(e) = smallest c >= 0 not used by any neighbour f < e, where   */
/* neighbours share at least one node.                                  */
/* ------------------------------------------------------------------ */
int oracle_colour(int dim, int64_t n_nodes, int64_t n_elems, const int32_t* conn,
                  const int32_t* ptr, const int32_t* ent, int32_t* colour, int32_t max_colours,
                  int32_t* n_colours) {
    (void)n_nodes;
    const int nv = dim + 1;
    unsigned char* used = (unsigned char*)calloc((size_t)max_colours + 1, 1);
    if (!used) return OR_ERR_CAPACITY;
    int32_t nc = 0;
    for (int64_t e = 0; e < n_elems; ++e) {
        memset(used, 0, (size_t)max_colours + 1);
        for (int a = 0; a < nv; ++a) {
            int32_t n = conn[e * nv + a];
            for (int32_t k = ptr[n]; k < ptr[n + 1]; ++k) {
                int64_t f = ent[k] / nv;
                if (f < e && colour[f] <= max_colours) used[colour[f]] = 1;
            }
        }
        int32_t c = 0;
        while (c < max_colours && used[c]) ++c;
        if (c >= max_colours) { free(used); g_err_index = e; return OR_ERR_CAPACITY; }
        colour[e] = c;
        if (c + 1 > nc) nc = c + 1;
    }
    free(used);
    *n_colours = nc;
    return OR_OK;
}

/* colour_elems sorted by (colour, element); colour_ptr[c] offsets */
int oracle_colour_sort(int64_t n_elems, const int32_t* colour, int32_t n_colours,
                       int32_t* colour_elems, int32_t* colour_ptr) {
    for (int32_t c = 0; c <= n_colours; ++c) colour_ptr[c] = 0;
    for (int64_t e = 0; e < n_elems; ++e) colour_ptr[colour[e] + 1] += 1;
    for (int32_t c = 0; c < n_colours; ++c) colour_ptr[c + 1] += colour_ptr[c];
    int32_t* fill = (int32_t*)calloc((size_t)n_colours, sizeof(int32_t));
    if (!fill) return OR_ERR_CAPACITY;
    for (int64_t e = 0; e < n_elems; ++e) {
        int32_t c = colour[e];
        colour_elems[colour_ptr[c] + fill[c]++] = (int32_t)e;
    }
    free(fill);
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Kinematics: F = I + grad u, grad u = sum_{a=0..d} u_a (x) */
/* grad N_a  (x = N_I x_I)                                 */
/* ------------------------------------------------------------------ */
static void elem_F(int dim, const int32_t* c, const double* u, double g[4][3], double F[3][3]) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) F[i][j] = (i == j) ? 1.0 : 0.0;
    for (int a = 0; a <= dim; ++a)
        for (int i = 0; i < dim; ++i)
            for (int j = 0; j < dim; ++j) F[i][j] += u[(int64_t)c[a] * dim + i] * g[a][j];
}

/* Voigt strain-displacement matrix B (small strain), engineering shear.
 * 3-D rows: eps11, eps22, eps33, 2eps23, 2eps13, 2eps12; 2-D: eps11, eps22, 2eps12.
 * Column index a*d + i.                                               */
static int voigt_B(int dim, double g[4][3], double B[6][12]) {
    const int nv = dim + 1;
    memset(B, 0, sizeof(double) * 6 * 12);
    if (dim == 2) {
        for (int a = 0; a < nv; ++a) {
            B[0][a * 2 + 0] = g[a][0];
            B[1][a * 2 + 1] = g[a][1];
            B[2][a * 2 + 0] = g[a][1];
            B[2][a * 2 + 1] = g[a][0];
        }
        return 3;
    }
    for (int a = 0; a < nv; ++a) {
        B[0][a * 3 + 0] = g[a][0];
        B[1][a * 3 + 1] = g[a][1];
        B[2][a * 3 + 2] = g[a][2];
        B[3][a * 3 + 1] = g[a][2];
        B[3][a * 3 + 2] = g[a][1];
        B[4][a * 3 + 0] = g[a][2];
        B[4][a * 3 + 2] = g[a][0];
        B[5][a * 3 + 0] = g[a][1];
        B[5][a * 3 + 1] = g[a][0];
    }
    return 6;
}

/* isotropic elasticity matrix D (Voigt, engineering shear): sigma = 2 mu eps + lam tr(eps) I,
 * written with the paper's coefficients 2mu = E/(1+nu), lam = E nu/((1+nu)(1-2nu));
 * 2-D is plane strain (reading R1).                                    */
static void voigt_D(int dim, double mu, double lam, double D[6][6]) {
    memset(D, 0, sizeof(double) * 36);
    int nn = dim;             /* normal components */
    int ns = dim == 2 ? 1 : 3;
    for (int i = 0; i < nn; ++i)
        for (int j = 0; j < nn; ++j) D[i][j] = lam + (i == j ? 2.0 * mu : 0.0);
    for (int k = 0; k < ns; ++k) D[nn + k][nn + k] = mu;
}

/* Voigt index pairs */
static const int VI3[6][2] = {{0, 0}, {1, 1}, {2, 2}, {1, 2}, {0, 2}, {0, 1}};
static const int VI2[3][2] = {{0, 0}, {1, 1}, {0, 1}};

/* Neo-Hookean second Piola-Kirchhoff stress and tangent (App. B; from Psi of P:713-722):
 * S = mu (I - C^{-1}) + lam ln J C^{-1};
 * C^SE_IJKL = lam Ci_IJ Ci_KL + (mu - lam ln J)(Ci_IK Ci_JL + Ci_IL Ci_JK).   */
static int nh_state(int dim, double F[3][3], double mu, double lam, double S[3][3],
                    double Ci[3][3], double* J_out, double* lnJ_out, double* psi_out) {
    double C[3][3] = {{0}};
    for (int I = 0; I < dim; ++I)
        for (int Jx = 0; Jx < dim; ++Jx)
            for (int k = 0; k < dim; ++k) C[I][Jx] += F[k][I] * F[k][Jx];
    double Fd[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Fd[i][j] = F[i][j];
    double J = dim == 2 ? (Fd[0][0] * Fd[1][1] - Fd[0][1] * Fd[1][0]) : det3(Fd);
    if (!(J > 0.0)) {
        /* inverted element (reading R3): every output is NaN, never left uninitialised */
        for (int I = 0; I < 3; ++I)
            for (int Jx = 0; Jx < 3; ++Jx) S[I][Jx] = Ci[I][Jx] = NAN;
        *J_out = J;
        *lnJ_out = NAN;
        *psi_out = NAN;
        return OR_ERR_INVERTED;
    }
    double lnJ = log(J);
    double I1 = 0.0;
    for (int i = 0; i < dim; ++i) I1 += C[i][i];
    inv_dd(dim, C, Ci);
    for (int I = 0; I < dim; ++I)
        for (int Jx = 0; Jx < dim; ++Jx)
            S[I][Jx] = mu * ((I == Jx ? 1.0 : 0.0) - Ci[I][Jx]) + lam * lnJ * Ci[I][Jx];
    *J_out = J;
    *lnJ_out = lnJ;
    *psi_out = 0.5 * lam * lnJ * lnJ - mu * lnJ + 0.5 * mu * (I1 - (double)dim);
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Element energy W_e = V_e Psi_e; totals W_{s,k} = sum_{e in part k} W_e; */
/* optional Pi = W - sum_{n in part k} f_ext,n . u_n */
/* ------------------------------------------------------------------ */
int oracle_energy(int dim, int64_t n_nodes, int64_t n_elems, const int32_t* conn,
                  const double* grad, const double* vol, int model, const double* mu,
                  const double* lam, int n_samples, const double* u, int n_parts,
                  const int32_t* part_elem, const int32_t* part_node, const double* f_ext,
                  double* W_e, double* totals) {
    const int nv = dim + 1;
    double* W = W_e ? W_e : (double*)malloc(sizeof(double) * (size_t)n_elems * n_samples);
    if (!W) return OR_ERR_CAPACITY;
    int64_t first_bad = -1;
    for (int s = 0; s < n_samples; ++s) {
        const double* us = u + (int64_t)s * n_nodes * dim;
        double* Ws = W + (int64_t)s * n_elems;
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < n_elems; ++e) {
            double g[4][3];
            elem_grads(dim, grad, e, g);
            const int32_t* c = conn + e * nv;
            double psi;
            if (model == OR_LINEAR) {
                double B[6][12], D[6][6], eps[6] = {0}, sig[6] = {0};
                int nvo = voigt_B(dim, g, B);
                voigt_D(dim, mu[e], lam[e], D);
                for (int r = 0; r < nvo; ++r)
                    for (int a = 0; a < nv; ++a)
                        for (int i = 0; i < dim; ++i)
                            eps[r] += B[r][a * dim + i] * us[(int64_t)c[a] * dim + i];
                for (int r = 0; r < nvo; ++r)
                    for (int q = 0; q < nvo; ++q) sig[r] += D[r][q] * eps[q];
                psi = 0.0;
                for (int r = 0; r < nvo; ++r) psi += 0.5 * sig[r] * eps[r];   /* 1/2 sigma:eps */
            } else {
                double F[3][3], S[3][3], Ci[3][3], J, lnJ;
                elem_F(dim, c, us, g, F);
                if (nh_state(dim, F, mu[e], lam[e], S, Ci, &J, &lnJ, &psi) != OR_OK) {
#pragma omp critical
                    { if (first_bad < 0 || e < first_bad) first_bad = e; }
                    psi = NAN;
                }
            }
            Ws[e] = vol[e] * psi;
        }
    }
    for (int s = 0; s < n_samples; ++s) {
        const double* us = u + (int64_t)s * n_nodes * dim;
        for (int k = 0; k < n_parts; ++k) {
            double acc = 0.0;
            for (int64_t e = part_elem[k]; e < part_elem[k + 1]; ++e) acc += W[(int64_t)s * n_elems + e];
            if (f_ext) {
                double work = 0.0;
                for (int64_t n = part_node[k]; n < part_node[k + 1]; ++n)
                    for (int i = 0; i < dim; ++i) work += f_ext[n * dim + i] * us[n * dim + i];
                acc -= work;
            }
            totals[(int64_t)s * n_parts + k] = acc;
        }
    }
    if (!W_e) free(W);
    if (first_bad >= 0) { g_err_index = first_bad; return OR_ERR_INVERTED; }
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Internal force (residual without f_ext; reading R7):                 */
/*  linear: f_e = V B^T D B u_e (virtual power)            */
/*  NH:     f_iI = V dN_I/dX_l F_ik S_kl (total Lagrangian) */
/* assembled sequentially in ascending (e, a) order.                    */
/* ------------------------------------------------------------------ */
int oracle_residual(int dim, int64_t n_nodes, int64_t n_elems, const int32_t* conn,
                    const double* grad, const double* vol, int model, const double* mu,
                    const double* lam, int n_samples, const double* u, double* r) {
    const int nv = dim + 1;
    const int ne = nv * dim;
    double* fe = (double*)malloc(sizeof(double) * (size_t)n_elems * ne);
    if (!fe) return OR_ERR_CAPACITY;
    int64_t first_bad = -1;
    for (int s = 0; s < n_samples; ++s) {
        const double* us = u + (int64_t)s * n_nodes * dim;
        double* rs = r + (int64_t)s * n_nodes * dim;
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < n_elems; ++e) {
            double g[4][3];
            elem_grads(dim, grad, e, g);
            const int32_t* c = conn + e * nv;
            double* f = fe + e * ne;
            if (model == OR_LINEAR) {
                double B[6][12], D[6][6], eps[6] = {0}, sig[6] = {0};
                int nvo = voigt_B(dim, g, B);
                voigt_D(dim, mu[e], lam[e], D);
                for (int q = 0; q < nvo; ++q)
                    for (int a = 0; a < nv; ++a)
                        for (int i = 0; i < dim; ++i)
                            eps[q] += B[q][a * dim + i] * us[(int64_t)c[a] * dim + i];
                for (int q = 0; q < nvo; ++q)
                    for (int p = 0; p < nvo; ++p) sig[q] += D[q][p] * eps[p];
                for (int k = 0; k < ne; ++k) {
                    double acc = 0.0;
                    for (int q = 0; q < nvo; ++q) acc += B[q][k] * sig[q];
                    f[k] = vol[e] * acc;
                }
            } else {
                double F[3][3], S[3][3], Ci[3][3], J, lnJ, psi;
                elem_F(dim, c, us, g, F);
                if (nh_state(dim, F, mu[e], lam[e], S, Ci, &J, &lnJ, &psi) != OR_OK) {
#pragma omp critical
                    { if (first_bad < 0 || e < first_bad) first_bad = e; }
                }
                for (int a = 0; a < nv; ++a)
                    for (int i = 0; i < dim; ++i) {
                        double acc = 0.0;
                        for (int k = 0; k < dim; ++k)
                            for (int l = 0; l < dim; ++l) acc += g[a][l] * F[i][k] * S[k][l];
                        f[a * dim + i] = vol[e] * acc;
                    }
            }
        }
        for (int64_t k = 0; k < n_nodes * dim; ++k) rs[k] = 0.0;
        for (int64_t e = 0; e < n_elems; ++e)
            for (int a = 0; a < nv; ++a)
                for (int i = 0; i < dim; ++i)
                    rs[(int64_t)conn[e * nv + a] * dim + i] += fe[e * ne + a * dim + i];
    }
    free(fe);
    if (first_bad >= 0) { g_err_index = first_bad; return OR_ERR_INVERTED; }
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Element tangent matrix K_e (ne x ne, row/col index a*d + i):          */
/*  linear: V B^T D B;  NH: V (G0^T S G0 + B0^T C^SE B0)  */
/* ------------------------------------------------------------------ */
/* The factors of the element tangent: strain-displacement matrix B (linear: Voigt B; NH: B0(F)),
 * material matrix D (linear: Voigt D; NH: C^SE in Voigt form) and, for NH, the second
 * Piola-Kirchhoff stress S of the geometric term (zero for linear).  Returns the status of the
 * NH state (OR_ERR_INVERTED for J <= 0, all factors NaN). */
static int tangent_factors(int dim, int model, double g[4][3], double mu, double lam, const int32_t* c,
                           const double* us, double B[6][12], double D[6][6], double S[3][3], int* nvo_out) {
    const int nv = dim + 1;
    if (model == OR_LINEAR) {
        *nvo_out = voigt_B(dim, g, B);
        voigt_D(dim, mu, lam, D);
        memset(S, 0, sizeof(double) * 9);
        return OR_OK;
    }
    double F[3][3], Ci[3][3], J, lnJ, psi;
    elem_F(dim, c, us, g, F);
    int st = nh_state(dim, F, mu, lam, S, Ci, &J, &lnJ, &psi);
    const int nvo = dim == 2 ? 3 : 6;
    const int (*VI)[2] = dim == 2 ? VI2 : VI3;
    /* C^SE in Voigt form (engineering shear for strains) */
    for (int x = 0; x < nvo; ++x)
        for (int y = 0; y < nvo; ++y) {
            int I = VI[x][0], Jx = VI[x][1], K2 = VI[y][0], L = VI[y][1];
            D[x][y] = lam * Ci[I][Jx] * Ci[K2][L] + (mu - lam * lnJ) * (Ci[I][K2] * Ci[Jx][L] + Ci[I][L] * Ci[Jx][K2]);
        }
    /* B0: delta E (Voigt, engineering shear) = B0 delta u;
     * dE_KL = 1/2 (F_iK dN_a/dX_L + F_iL dN_a/dX_K) du_ia, shear rows doubled. */
    memset(B, 0, sizeof(double) * 6 * 12);
    for (int x = 0; x < nvo; ++x) {
        int Kk = VI[x][0], L = VI[x][1];
        for (int a = 0; a < nv; ++a)
            for (int i = 0; i < dim; ++i) {
                double v = (Kk == L) ? F[i][Kk] * g[a][L]
                                     : F[i][Kk] * g[a][L] + F[i][L] * g[a][Kk];
                B[x][a * dim + i] = v;
            }
    }
    *nvo_out = nvo;
    return st;
}

static int elem_tangent(int dim, int model, double g[4][3], double V, double mu, double lam,
                        const int32_t* c, const double* us, double K[12][12]) {
    const int nv = dim + 1, ne = nv * dim;
    double B[6][12], D[6][6], S[3][3];
    int nvo = 0;
    int st = tangent_factors(dim, model, g, mu, lam, c, us, B, D, S, &nvo);
    memset(K, 0, sizeof(double) * 144);
    for (int p = 0; p < ne; ++p)
        for (int q = 0; q < ne; ++q) {
            double acc = 0.0;
            for (int x = 0; x < nvo; ++x)
                for (int y = 0; y < nvo; ++y) acc += B[x][p] * D[x][y] * B[y][q];
            K[p][q] = V * acc;
        }
    if (model == OR_LINEAR) return st;
    /* geometric: K_geo[(a,i),(b,j)] = delta_ij grad N_a . S . grad N_b */
    for (int a = 0; a < nv; ++a)
        for (int b = 0; b < nv; ++b) {
            double gsg = 0.0;
            for (int k = 0; k < dim; ++k)
                for (int l = 0; l < dim; ++l) gsg += g[a][k] * S[k][l] * g[b][l];
            for (int i = 0; i < dim; ++i) K[a * dim + i][b * dim + i] += V * gsg;
        }
    return st;
}

/* K_e v_e without forming K_e: the same product V (B^T D B + G0^T S G0) v_e evaluated right to
 * left, B^T (D (B v_e)) (reading R30: the association order of the matrix chain) */
static int elem_tangent_apply(int dim, int model, double g[4][3], double V, double mu, double lam,
                              const int32_t* c, const double* us, const double* ve, double* out) {
    const int nv = dim + 1, ne = nv * dim;
    double B[6][12], D[6][6], S[3][3], eps[6], sig[6];
    int nvo = 0;
    int st = tangent_factors(dim, model, g, mu, lam, c, us, B, D, S, &nvo);
    for (int x = 0; x < nvo; ++x) {
        double acc = 0.0;
        for (int q = 0; q < ne; ++q) acc += B[x][q] * ve[q];
        eps[x] = acc;
    }
    for (int x = 0; x < nvo; ++x) {
        double acc = 0.0;
        for (int y = 0; y < nvo; ++y) acc += D[x][y] * eps[y];
        sig[x] = acc;
    }
    for (int p = 0; p < ne; ++p) {
        double acc = 0.0;
        for (int x = 0; x < nvo; ++x) acc += B[x][p] * sig[x];
        out[p] = V * acc;
    }
    if (model == OR_LINEAR) return st;
    /* geometric: (K_geo v)_(a,i) = sum_b (grad N_a . S . grad N_b) v_(b,i) */
    for (int a = 0; a < nv; ++a)
        for (int b = 0; b < nv; ++b) {
            double gsg = 0.0;
            for (int k = 0; k < dim; ++k)
                for (int l = 0; l < dim; ++l) gsg += g[a][k] * S[k][l] * g[b][l];
            for (int i = 0; i < dim; ++i) out[a * dim + i] += V * gsg * ve[b * dim + i];
        }
    return st;
}

/* association of the element product: 0 = B^T (D (B v_e)) (default), 1 = (B^T D B) v_e with the
 * element matrix formed first.  Form 1 exists only to widen the oracle's own CG iteration-count
 * spread over valid orderings of the same sums (reading R18). */
static int g_tangent_form = 0;
void oracle_set_tangent_form(int form) { g_tangent_form = form; }

/* ------------------------------------------------------------------ */
/* Matrix-free tangent apply with optional Dirichlet mask (reading R9):  */
/*   A v = (I - M) K (I - M) v + M v                                      */
/* u: NH state [S][N][d] (ignored for linear, may be NULL)                */
/* ------------------------------------------------------------------ */
int oracle_tangent(int dim, int64_t n_nodes, int64_t n_elems, const int32_t* conn,
                   const double* grad, const double* vol, int model, const double* mu,
                   const double* lam, int n_samples, const double* u, const double* v,
                   const uint8_t* mask, double* Kv) {
    const int nv = dim + 1, ne = nv * dim;
    double* fe = (double*)malloc(sizeof(double) * (size_t)n_elems * ne);
    if (!fe) return OR_ERR_CAPACITY;
    int64_t first_bad = -1;
    for (int s = 0; s < n_samples; ++s) {
        const double* vs = v + (int64_t)s * n_nodes * dim;
        const double* us = u ? u + (int64_t)s * n_nodes * dim : NULL;
        double* out = Kv + (int64_t)s * n_nodes * dim;
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < n_elems; ++e) {
            double g[4][3], ve[12];
            elem_grads(dim, grad, e, g);
            const int32_t* c = conn + e * nv;
            for (int a = 0; a < nv; ++a)
                for (int i = 0; i < dim; ++i) {
                    int64_t dof = (int64_t)c[a] * dim + i;
                    ve[a * dim + i] = (mask && mask[dof]) ? 0.0 : vs[dof];
                }
            int est;
            if (g_tangent_form == 1) {
                /* formed element matrix, then K_e v_e (the other association of the same chain) */
                double K[12][12];
                est = elem_tangent(dim, model, g, vol[e], mu[e], lam[e], c, us, K);
                for (int p = 0; p < ne; ++p) {
                    double acc = 0.0;
                    for (int q = 0; q < ne; ++q) acc += K[p][q] * ve[q];
                    fe[e * ne + p] = acc;
                }
            } else {
                est = elem_tangent_apply(dim, model, g, vol[e], mu[e], lam[e], c, us, ve, fe + e * ne);
            }
            if (est != OR_OK) {
#pragma omp critical
                { if (first_bad < 0 || e < first_bad) first_bad = e; }
            }
        }
        for (int64_t k = 0; k < n_nodes * dim; ++k) out[k] = 0.0;
        for (int64_t e = 0; e < n_elems; ++e)
            for (int a = 0; a < nv; ++a)
                for (int i = 0; i < dim; ++i)
                    out[(int64_t)conn[e * nv + a] * dim + i] += fe[e * ne + a * dim + i];
        if (mask)
            for (int64_t k = 0; k < n_nodes * dim; ++k)
                if (mask[k]) out[k] = vs[k];
    }
    free(fe);
    if (first_bad >= 0) { g_err_index = first_bad; return OR_ERR_INVERTED; }
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Warm-started CG (App. B; warm start P:395-417; skip rule P:419-423) */
/* Solves A x = b with A = (I-M)K(I-M) + M, b = (I-M)(f - K x_D) + M x0, x_D = M x0 */
/* (reading R9/R10).  Hestenes-Stiefel, unpreconditioned, stop on the   */
/* recurrence residual ||r|| < tol ||b_free|| (reading R8), k = number of */
/* A p products in the loop (reading R11).                               */
/* ------------------------------------------------------------------ */
/* dot product; order 0: sequential ascending (default), 1: sequential descending,
 * 2: pairwise (recursive halving), 3: blocked (sums of 1024-term ascending blocks),
 * 4: compensated (Kahan).  Orders 1-4 exist only to measure the oracle's own
 * iteration-count spread under valid re-orderings of the sums (reading R18). */
static int g_dot_order = 0;

static double dot_pairwise(int64_t n, const double* a, const double* b) {
    if (n <= 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
        return s;
    }
    int64_t h = n / 2;
    return dot_pairwise(h, a, b) + dot_pairwise(n - h, a + h, b + h);
}

static double dot(int64_t n, const double* a, const double* b) {
    double s = 0.0;
    if (g_dot_order == 1) {
        for (int64_t i = n - 1; i >= 0; --i) s += a[i] * b[i];
        return s;
    }
    if (g_dot_order == 2) return dot_pairwise(n, a, b);
    if (g_dot_order == 3) {
        for (int64_t i0 = 0; i0 < n; i0 += 1024) {
            double t = 0.0;
            for (int64_t i = i0; i < n && i < i0 + 1024; ++i) t += a[i] * b[i];
            s += t;
        }
        return s;
    }
    if (g_dot_order == 4) {
        double c = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double y = a[i] * b[i] - c;
            double t = s + y;
            c = (t - s) - y;
            s = t;
        }
        return s;
    }
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

void oracle_set_dot_order(int order) { g_dot_order = order; }

/* one dot product under a given order (exported so the orders can be pinned against an exact
 * dot product: tests/test_oracle_pins.py) */
double oracle_dot(int order, int64_t n, const double* a, const double* b) {
    const int saved = g_dot_order;
    g_dot_order = order;
    const double s = dot(n, a, b);
    g_dot_order = saved;
    return s;
}

/* the operator of a CG solve: out = K v, or (I-M) K (I-M) v + M v when mask != NULL */
typedef int (*or_apply)(void* ctx, const double* v, const uint8_t* mask, double* out);

struct simplex_op {
    int dim; int64_t n_nodes, n_elems; const int32_t* conn; const double* grad; const double* vol;
    int model; const double* mu; const double* lam; const double* u_state;
};
static int simplex_apply(void* ctx, const double* v, const uint8_t* mask, double* out) {
    const struct simplex_op* o = (const struct simplex_op*)ctx;
    return oracle_tangent(o->dim, o->n_nodes, o->n_elems, o->conn, o->grad, o->vol, o->model, o->mu, o->lam, 1,
                          o->u_state, v, mask, out);
}

/* Hestenes-Stiefel CG on the masked operator A (App. B, reading R8-R11) */
static int cg_core(int64_t n, or_apply A, void* ctx, const double* f, const uint8_t* mask, double* x, double tol,
                   int32_t max_iter, double* history, int32_t* iterations, double* rel_res0,
                   double* rel_res_final, double* true_rel_res_final) {
    double* r = (double*)malloc(sizeof(double) * n);
    double* p = (double*)malloc(sizeof(double) * n);
    double* q = (double*)malloc(sizeof(double) * n);
    double* xd = (double*)malloc(sizeof(double) * n);
    double* b = (double*)malloc(sizeof(double) * n);
    if (!r || !p || !q || !xd || !b) return OR_ERR_CAPACITY;
    int st = OR_OK;
    /* b = (I - M)(f - K x_D): K x_D via the unmasked operator */
    for (int64_t i = 0; i < n; ++i) xd[i] = (mask && mask[i]) ? x[i] : 0.0;
    A(ctx, xd, NULL, q);
    for (int64_t i = 0; i < n; ++i) b[i] = (mask && mask[i]) ? 0.0 : f[i] - q[i];
    double bnorm = sqrt(dot(n, b, b));
    /* r = b - A x over free DOFs (constrained rows of A x - (M x0) vanish) */
    A(ctx, x, mask, q);
    for (int64_t i = 0; i < n; ++i) r[i] = (mask && mask[i]) ? 0.0 : b[i] - q[i];
    double rho = dot(n, r, r);
    *iterations = 0;
    *rel_res0 = bnorm > 0 ? sqrt(rho) / bnorm : 0.0;
    if (history) history[0] = *rel_res0;
    int32_t k = 0;
    if (bnorm == 0.0) {
        for (int64_t i = 0; i < n; ++i) x[i] = (mask && mask[i]) ? x[i] : 0.0;
        *rel_res_final = 0.0;
        rho = 0.0;
    } else if (sqrt(rho) < tol * bnorm) {
        /* skip rule: the supplied guess already satisfies the test */
    } else {
        memcpy(p, r, sizeof(double) * n);
        st = OR_ERR_NOT_CONVERGED;
        for (k = 1; k <= max_iter; ++k) {
            A(ctx, p, mask, q);
            double pi = dot(n, p, q);
            if (!(pi > 0.0)) { st = OR_ERR_BREAKDOWN; break; }
            double alpha = rho / pi;
            for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
            for (int64_t i = 0; i < n; ++i) r[i] -= alpha * q[i];
            double rho_new = dot(n, r, r);
            if (history) history[k] = sqrt(rho_new) / bnorm;
            if (sqrt(rho_new) < tol * bnorm) { rho = rho_new; st = OR_OK; break; }
            double beta = rho_new / rho;
            for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
            rho = rho_new;
        }
        if (k > max_iter) k = max_iter;
    }
    *iterations = k;
    *rel_res_final = bnorm > 0 ? sqrt(rho) / bnorm : 0.0;
    /* true residual ||b - A x|| / ||b|| over free DOFs */
    A(ctx, x, mask, q);
    double tr = 0.0;
    for (int64_t i = 0; i < n; ++i)
        if (!(mask && mask[i])) tr += (b[i] - q[i]) * (b[i] - q[i]);
    *true_rel_res_final = bnorm > 0 ? sqrt(tr) / bnorm : 0.0;
    free(r); free(p); free(q); free(xd); free(b);
    return st;
}

int oracle_cg(int dim, int64_t n_nodes, int64_t n_elems, const int32_t* conn, const double* grad,
              const double* vol, int model, const double* mu, const double* lam,
              const double* u_state, const double* f, const uint8_t* mask, double* x, double tol,
              int32_t max_iter, double* history, int32_t* iterations, double* rel_res0,
              double* rel_res_final, double* true_rel_res_final) {
    struct simplex_op o = {dim, n_nodes, n_elems, conn, grad, vol, model, mu, lam, u_state};
    return cg_core(n_nodes * dim, simplex_apply, &o, f, mask, x, tol, max_iter, history, iterations, rel_res0,
                   rel_res_final, true_rel_res_final);
}

/* ------------------------------------------------------------------ */
/* Jacobi preconditioner (the paper sets preconditioning beside warm  */
/* starting as a complementary way to cut CG iterations, §5.5):                  */
/*   diag[k] = A_kk of A = (I-M) K(u) (I-M) + M, i.e. the sum over the (e, a) entries of   */
/*   node n of the diagonal entries K_e[a*d+i][a*d+i] of the textbook element tangent      */
/*   (Voigt B^T D B / V (G0^T S G0 + B0^T C^SE B0), elem_tangent above), assembled in      */
/*   ascending (e, a) order; 1 on constrained DOFs.                                        */
/* ------------------------------------------------------------------ */
int oracle_tangent_diag(int dim, int64_t n_nodes, int64_t n_elems, const int32_t* conn,
                        const double* grad, const double* vol, int model, const double* mu,
                        const double* lam, const double* u, const uint8_t* mask, double* diag) {
    const int nv = dim + 1, ne = nv * dim;
    double* de = (double*)malloc(sizeof(double) * (size_t)n_elems * ne);
    if (!de) return OR_ERR_CAPACITY;
    int64_t first_bad = -1;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n_elems; ++e) {
        double g[4][3], K[12][12];
        elem_grads(dim, grad, e, g);
        if (elem_tangent(dim, model, g, vol[e], mu[e], lam[e], conn + e * nv, u, K) != OR_OK) {
#pragma omp critical
            { if (first_bad < 0 || e < first_bad) first_bad = e; }
        }
        for (int p = 0; p < ne; ++p) de[e * ne + p] = K[p][p];
    }
    for (int64_t k = 0; k < n_nodes * dim; ++k) diag[k] = 0.0;
    for (int64_t e = 0; e < n_elems; ++e)
        for (int a = 0; a < nv; ++a)
            for (int i = 0; i < dim; ++i) diag[(int64_t)conn[e * nv + a] * dim + i] += de[e * ne + a * dim + i];
    if (mask)
        for (int64_t k = 0; k < n_nodes * dim; ++k)
            if (mask[k]) diag[k] = 1.0;
    free(de);
    if (first_bad >= 0) { g_err_index = first_bad; return OR_ERR_INVERTED; }
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Preconditioned CG (textbook Hestenes-Stiefel PCG with M^-1 = diag(A)^-1, reading R27):   */
/*   r0 = b - A x0 (free DOFs), z0 = M^-1 r0, p0 = z0, rho = r.z                             */
/*   q = A p; pi = p.q; alpha = rho / pi; x += alpha p; r -= alpha q                          */
/*   stop when ||r|| < tol ||b_free|| (the same unpreconditioned test as oracle_cg, R8)       */
/*   z = M^-1 r; rho' = r.z; beta = rho' / rho; p = z + beta p                               */
/* M^-1_k = 1 / diag_k where diag_k > 0, else 1.  precond 0 runs plain CG (z = r).           */
/* ------------------------------------------------------------------ */
int oracle_pcg(int dim, int64_t n_nodes, int64_t n_elems, const int32_t* conn, const double* grad,
               const double* vol, int model, const double* mu, const double* lam,
               const double* u_state, const double* f, const uint8_t* mask, int precond, double* x,
               double tol, int32_t max_iter, double* history, int32_t* iterations, double* rel_res0,
               double* rel_res_final, double* true_rel_res_final) {
    const int64_t n = n_nodes * dim;
    double* r = (double*)malloc(sizeof(double) * n);
    double* z = (double*)malloc(sizeof(double) * n);
    double* p = (double*)malloc(sizeof(double) * n);
    double* q = (double*)malloc(sizeof(double) * n);
    double* xd = (double*)malloc(sizeof(double) * n);
    double* b = (double*)malloc(sizeof(double) * n);
    double* minv = (double*)malloc(sizeof(double) * n);
    if (!r || !z || !p || !q || !xd || !b || !minv) return OR_ERR_CAPACITY;
    int st = OR_OK;
    if (precond) {
        oracle_tangent_diag(dim, n_nodes, n_elems, conn, grad, vol, model, mu, lam, u_state, mask, minv);
        for (int64_t i = 0; i < n; ++i) minv[i] = minv[i] > 0.0 ? 1.0 / minv[i] : 1.0;
    } else {
        for (int64_t i = 0; i < n; ++i) minv[i] = 1.0;
    }
    for (int64_t i = 0; i < n; ++i) xd[i] = (mask && mask[i]) ? x[i] : 0.0;
    oracle_tangent(dim, n_nodes, n_elems, conn, grad, vol, model, mu, lam, 1, u_state, xd, NULL, q);
    for (int64_t i = 0; i < n; ++i) b[i] = (mask && mask[i]) ? 0.0 : f[i] - q[i];
    double bnorm = sqrt(dot(n, b, b));
    oracle_tangent(dim, n_nodes, n_elems, conn, grad, vol, model, mu, lam, 1, u_state, x, mask, q);
    for (int64_t i = 0; i < n; ++i) r[i] = (mask && mask[i]) ? 0.0 : b[i] - q[i];
    double rr = dot(n, r, r);
    *rel_res0 = bnorm > 0 ? sqrt(rr) / bnorm : 0.0;
    if (history) history[0] = *rel_res0;
    int32_t k = 0;
    if (bnorm == 0.0) {
        for (int64_t i = 0; i < n; ++i) x[i] = (mask && mask[i]) ? x[i] : 0.0;
        rr = 0.0;
    } else if (sqrt(rr) < tol * bnorm) {
        /* skip rule */
    } else {
        for (int64_t i = 0; i < n; ++i) z[i] = minv[i] * r[i];
        memcpy(p, z, sizeof(double) * n);
        double rho = dot(n, r, z);
        st = OR_ERR_NOT_CONVERGED;
        for (k = 1; k <= max_iter; ++k) {
            oracle_tangent(dim, n_nodes, n_elems, conn, grad, vol, model, mu, lam, 1, u_state, p, mask, q);
            double pi = dot(n, p, q);
            if (!(pi > 0.0)) { st = OR_ERR_BREAKDOWN; break; }
            double alpha = rho / pi;
            for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
            for (int64_t i = 0; i < n; ++i) r[i] -= alpha * q[i];
            rr = dot(n, r, r);
            if (history) history[k] = sqrt(rr) / bnorm;
            if (sqrt(rr) < tol * bnorm) { st = OR_OK; break; }
            for (int64_t i = 0; i < n; ++i) z[i] = minv[i] * r[i];
            double rho_new = dot(n, r, z);
            double beta = rho_new / rho;
            for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
            rho = rho_new;
        }
        if (k > max_iter) k = max_iter;
    }
    *iterations = k;
    *rel_res_final = bnorm > 0 ? sqrt(rr) / bnorm : 0.0;
    oracle_tangent(dim, n_nodes, n_elems, conn, grad, vol, model, mu, lam, 1, u_state, x, mask, q);
    double tr = 0.0;
    for (int64_t i = 0; i < n; ++i)
        if (!(mask && mask[i])) tr += (b[i] - q[i]) * (b[i] - q[i]);
    *true_rel_res_final = bnorm > 0 ? sqrt(tr) / bnorm : 0.0;
    free(r); free(z); free(p); free(q); free(xd); free(b); free(minv);
    return st;
}

/* OpenMP threads of the oracle's parallel loops (timing only: every result is independent of
 * the thread count, since the assembly sums run sequentially) */
#ifdef _OPENMP
#include <omp.h>
void oracle_set_threads(int n) { omp_set_num_threads(n > 0 ? n : omp_get_num_procs()); }
#else
void oracle_set_threads(int n) { (void)n; }
#endif

/* ------------------------------------------------------------------ */
/* Steady-state heat conduction, the paper's scalar example (Eq.          */
/* poisson_equation P:186-198 and its energy form P:249-284), on P1 elements:                  */
/*   grad T_e = sum_{a>=1} (T_a - T_0) grad N_a  (= sum_a T_a grad N_a, grad N_0 = -sum)         */
/*   W_e = 1/2 k_e V_e |grad T_e|^2                                                              */
/*   totals[s][k] = sum_{e in part k} W_e - sum_{n in part k} f_n T_n   (f: consistent nodal    */
/*                  loads of the source and the boundary flux, nullable)                        */
/*   r_n = sum_{(e,a): v_a(e) = n} k_e V_e grad T_e . grad N_a  (dW/dT_n; the tangent is r(v))  */
/* assembled sequentially in ascending (e, a) order.                                             */
/* ------------------------------------------------------------------ */
int oracle_heat(int dim, int64_t n_nodes, int64_t n_elems, const int32_t* conn, const double* grad,
                const double* vol, const double* k, int64_t k_stride, int n_samples, const double* T,
                int n_parts, const int32_t* part_elem, const int32_t* part_node, const double* f,
                double* W, double* totals, double* r) {
    const int nv = dim + 1;
    for (int s = 0; s < n_samples; ++s) {
        const double* Ts = T + (int64_t)s * n_nodes;
        double* rs = r ? r + (int64_t)s * n_nodes : NULL;
        if (rs)
            for (int64_t n = 0; n < n_nodes; ++n) rs[n] = 0.0;
        for (int p = 0; p < n_parts; ++p) {
            double tot = 0.0;
            for (int64_t e = part_elem[p]; e < part_elem[p + 1]; ++e) {
                double g[4][3], gT[3] = {0.0, 0.0, 0.0};
                elem_grads(dim, grad, e, g);
                const int32_t* c = conn + e * nv;
                /* difference form (as the kinematics, c1 item 2): a constant field gives 0 exactly */
                for (int a = 1; a < nv; ++a)
                    for (int j = 0; j < dim; ++j) gT[j] += (Ts[c[a]] - Ts[c[0]]) * g[a][j];
                double gg = 0.0;
                for (int j = 0; j < dim; ++j) gg += gT[j] * gT[j];
                const double ke = k[e * k_stride];
                const double w = 0.5 * ke * vol[e] * gg;
                if (W) W[(int64_t)s * n_elems + e] = w;
                tot += w;
                if (rs)
                    for (int a = 0; a < nv; ++a) {
                        double dg = 0.0;
                        for (int j = 0; j < dim; ++j) dg += gT[j] * g[a][j];
                        rs[c[a]] += ke * vol[e] * dg;
                    }
            }
            if (f)
                for (int64_t n = part_node[p]; n < part_node[p + 1]; ++n) tot -= f[n] * Ts[n];
            if (totals) totals[(int64_t)s * n_parts + p] = tot;
        }
    }
    return OR_OK;
}

/* ================================================================== */
/* Quadrilateral elements with Gauss quadrature:  */
/* Q4 bilinear (2x2 Gauss) and Q8 serendipity (3x3 Gauss), 2-D plane    */
/* strain, isoparametric (App. B: x = N_I x_I, X = N_I X_I), */
/* the same constitutive laws as the simplex functions (P:527-536,      */
/* P:709-722), each element integral evaluated by its Gauss rule: the   */
/* beam's 50 x 50 Q4 mesh (§4.2) and Cook's 30 x 30 Q8 serendipity */
/* mesh.  Reading R33: node order, rules.           */
/* ================================================================== */
#define OR_Q4 1
#define OR_Q8 2

static int quad_nv(int type) { return type == OR_Q4 ? 4 : 8; }

/* reference coordinates of the nodes: corners counter-clockwise from (-1,-1), then the midsides
 * (0,-1), (1,0), (0,1), (-1,0) (Q8 only) */
static const double QXI[8][2] = {{-1, -1}, {1, -1}, {1, 1}, {-1, 1}, {0, -1}, {1, 0}, {0, 1}, {-1, 0}};

/* shape functions N_a(xi, eta) and their reference derivatives dN[a][0] = dN_a/dxi,
 * dN[a][1] = dN_a/deta */
int oracle_quad_shape(int type, double xi, double eta, double* N, double* dN) {
    if (type == OR_Q4) {
        for (int a = 0; a < 4; ++a) {
            const double xa = QXI[a][0], ya = QXI[a][1];
            N[a] = 0.25 * (1.0 + xi * xa) * (1.0 + eta * ya);
            dN[2 * a + 0] = 0.25 * xa * (1.0 + eta * ya);
            dN[2 * a + 1] = 0.25 * ya * (1.0 + xi * xa);
        }
        return OR_OK;
    }
    if (type != OR_Q8) return OR_ERR_ARG;
    for (int a = 0; a < 4; ++a) {   /* corners: 1/4 (1 + xi xa)(1 + eta ya)(xi xa + eta ya - 1) */
        const double xa = QXI[a][0], ya = QXI[a][1];
        N[a] = 0.25 * (1.0 + xi * xa) * (1.0 + eta * ya) * (xi * xa + eta * ya - 1.0);
        dN[2 * a + 0] = 0.25 * xa * (1.0 + eta * ya) * (2.0 * xi * xa + eta * ya);
        dN[2 * a + 1] = 0.25 * ya * (1.0 + xi * xa) * (xi * xa + 2.0 * eta * ya);
    }
    for (int a = 4; a < 8; ++a) {
        const double xa = QXI[a][0], ya = QXI[a][1];
        if (xa == 0.0) {            /* 1/2 (1 - xi^2)(1 + eta ya) */
            N[a] = 0.5 * (1.0 - xi * xi) * (1.0 + eta * ya);
            dN[2 * a + 0] = -xi * (1.0 + eta * ya);
            dN[2 * a + 1] = 0.5 * ya * (1.0 - xi * xi);
        } else {                    /* 1/2 (1 + xi xa)(1 - eta^2) */
            N[a] = 0.5 * (1.0 + xi * xa) * (1.0 - eta * eta);
            dN[2 * a + 0] = 0.5 * xa * (1.0 - eta * eta);
            dN[2 * a + 1] = -eta * (1.0 + xi * xa);
        }
    }
    return OR_OK;
}

/* tensor-product Gauss-Legendre rule: 2 x 2 for Q4, 3 x 3 for Q8; points eta-major */
int oracle_quad_rule(int type, double* pts, double* w) {
    const double g2[2] = {-1.0 / sqrt(3.0), 1.0 / sqrt(3.0)}, w2[2] = {1.0, 1.0};
    const double g3[3] = {-sqrt(0.6), 0.0, sqrt(0.6)}, w3[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
    const int m = type == OR_Q4 ? 2 : 3;
    const double* g = type == OR_Q4 ? g2 : g3;
    const double* wg = type == OR_Q4 ? w2 : w3;
    int k = 0;
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i, ++k) {
            pts[2 * k] = g[i];
            pts[2 * k + 1] = g[j];
            w[k] = wg[i] * wg[j];
        }
    return k;
}

/* geometry at one quadrature point: J_ij = sum_a X_{a,i} dN_a/dxi_j, dN_a/dX = dN_a/dxi J^-1;
 * returns det J */
static double quad_qp(int type, const double* coords, const int32_t* c, double xi, double eta, double dNdX[8][2]) {
    const int nv = quad_nv(type);
    double N[8], dN[16];
    oracle_quad_shape(type, xi, eta, N, dN);
    double J[2][2] = {{0, 0}, {0, 0}};
    for (int a = 0; a < nv; ++a)
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) J[i][j] += coords[(int64_t)c[a] * 2 + i] * dN[2 * a + j];
    const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double Ji[2][2] = {{J[1][1] / det, -J[0][1] / det}, {-J[1][0] / det, J[0][0] / det}};
    for (int a = 0; a < nv; ++a)
        for (int k = 0; k < 2; ++k) dNdX[a][k] = dN[2 * a] * Ji[0][k] + dN[2 * a + 1] * Ji[1][k];
    return det;
}

/* smallest det J over every element's quadrature points (validity: > 0) */
int oracle_quad_check(int type, int64_t n_nodes, int64_t n_elems, const double* coords, const int32_t* conn,
                      double* min_det) {
    if (type != OR_Q4 && type != OR_Q8) return OR_ERR_ARG;
    const int nv = quad_nv(type);
    double pts[18], w[9];
    const int nq = oracle_quad_rule(type, pts, w);
    double m = INFINITY;
    int64_t bad = -1;
    for (int64_t e = 0; e < n_elems; ++e) {
        for (int a = 0; a < nv; ++a)
            if (conn[e * nv + a] < 0 || conn[e * nv + a] >= n_nodes) { g_err_index = e; return OR_ERR_ARG; }
        for (int q = 0; q < nq; ++q) {
            double dNdX[8][2];
            const double det = quad_qp(type, coords, conn + e * nv, pts[2 * q], pts[2 * q + 1], dNdX);
            if (det < m) m = det;
            if (!(det > 0.0) && bad < 0) bad = e;
        }
    }
    *min_det = m;
    if (bad >= 0) { g_err_index = bad; return OR_ERR_DEGENERATE; }
    return OR_OK;
}

/* Voigt B (eps11, eps22, 2 eps12) of a 2-D element with nv nodes, column a*2 + i */
static void quad_B(int nv, double g[8][2], double B[3][16]) {
    memset(B, 0, sizeof(double) * 3 * 16);
    for (int a = 0; a < nv; ++a) {
        B[0][2 * a + 0] = g[a][0];
        B[1][2 * a + 1] = g[a][1];
        B[2][2 * a + 0] = g[a][1];
        B[2][2 * a + 1] = g[a][0];
    }
}

/* F = I + sum_a u_a (x) grad N_a (isoparametric) */
static void quad_F(int nv, const int32_t* c, const double* u, double g[8][2], double F[3][3]) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) F[i][j] = (i == j) ? 1.0 : 0.0;
    for (int a = 0; a < nv; ++a)
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) F[i][j] += u[(int64_t)c[a] * 2 + i] * g[a][j];
}

/* element energy and internal force of one quadrature point, accumulated with weight wd = w det J */
static int quad_point(int nv, int model, double g[8][2], double wd, double mu, double lam, const int32_t* c,
                      const double* u, double* W, double* f) {
    if (model == OR_LINEAR) {
        double B[3][16], D[6][6], eps[3] = {0, 0, 0}, sig[3] = {0, 0, 0};
        quad_B(nv, g, B);
        voigt_D(2, mu, lam, D);
        for (int r = 0; r < 3; ++r)
            for (int a = 0; a < nv; ++a)
                for (int i = 0; i < 2; ++i) eps[r] += B[r][2 * a + i] * u[(int64_t)c[a] * 2 + i];
        for (int r = 0; r < 3; ++r)
            for (int q = 0; q < 3; ++q) sig[r] += D[r][q] * eps[q];
        if (W) {
            double psi = 0.0;
            for (int r = 0; r < 3; ++r) psi += 0.5 * sig[r] * eps[r];
            *W += wd * psi;
        }
        if (f)
            for (int k = 0; k < 2 * nv; ++k) {
                double acc = 0.0;
                for (int r = 0; r < 3; ++r) acc += B[r][k] * sig[r];
                f[k] += wd * acc;
            }
        return OR_OK;
    }
    double F[3][3], S[3][3], Ci[3][3], J, lnJ, psi;
    quad_F(nv, c, u, g, F);
    const int st = nh_state(2, F, mu, lam, S, Ci, &J, &lnJ, &psi);
    if (W) *W += wd * psi;
    if (f)
        for (int a = 0; a < nv; ++a)
            for (int i = 0; i < 2; ++i) {
                double acc = 0.0;
                for (int k = 0; k < 2; ++k)
                    for (int l = 0; l < 2; ++l) acc += g[a][l] * F[i][k] * S[k][l];
                f[2 * a + i] += wd * acc;
            }
    return st;
}

/* K_e v_e of one quadrature point (linear: B^T D B v; NH: B0^T C^SE B0 v + G0^T S G0 v), added
 * with weight wd */
static int quad_point_tangent(int nv, int model, double g[8][2], double wd, double mu, double lam,
                              const int32_t* c, const double* u, const double* ve, double* out) {
    double B[3][16], D[6][6], S[3][3] = {{0}};
    int st = OR_OK;
    if (model == OR_LINEAR) {
        quad_B(nv, g, B);
        voigt_D(2, mu, lam, D);
    } else {
        double F[3][3], Ci[3][3], J, lnJ, psi;
        quad_F(nv, c, u, g, F);
        st = nh_state(2, F, mu, lam, S, Ci, &J, &lnJ, &psi);
        for (int x = 0; x < 3; ++x)
            for (int y = 0; y < 3; ++y) {
                int I = VI2[x][0], Jx = VI2[x][1], K2 = VI2[y][0], L = VI2[y][1];
                D[x][y] = lam * Ci[I][Jx] * Ci[K2][L] + (mu - lam * lnJ) * (Ci[I][K2] * Ci[Jx][L] + Ci[I][L] * Ci[Jx][K2]);
            }
        memset(B, 0, sizeof(B));
        for (int x = 0; x < 3; ++x) {
            int Kk = VI2[x][0], L = VI2[x][1];
            for (int a = 0; a < nv; ++a)
                for (int i = 0; i < 2; ++i)
                    B[x][2 * a + i] = (Kk == L) ? F[i][Kk] * g[a][L] : F[i][Kk] * g[a][L] + F[i][L] * g[a][Kk];
        }
    }
    double eps[3], sig[3];
    for (int x = 0; x < 3; ++x) {
        double acc = 0.0;
        for (int q = 0; q < 2 * nv; ++q) acc += B[x][q] * ve[q];
        eps[x] = acc;
    }
    for (int x = 0; x < 3; ++x) {
        double acc = 0.0;
        for (int y = 0; y < 3; ++y) acc += D[x][y] * eps[y];
        sig[x] = acc;
    }
    for (int p = 0; p < 2 * nv; ++p) {
        double acc = 0.0;
        for (int x = 0; x < 3; ++x) acc += B[x][p] * sig[x];
        out[p] += wd * acc;
    }
    if (model != OR_LINEAR)
        for (int a = 0; a < nv; ++a)
            for (int b = 0; b < nv; ++b) {
                double gsg = 0.0;
                for (int k = 0; k < 2; ++k)
                    for (int l = 0; l < 2; ++l) gsg += g[a][k] * S[k][l] * g[b][l];
                for (int i = 0; i < 2; ++i) out[2 * a + i] += wd * gsg * ve[2 * b + i];
            }
    return st;
}

/* energy, internal force and tangent of Q4 / Q8 meshes: element integrals by the Gauss rule,
 * per-element outputs, node sums sequential in ascending (element, node) order (as the simplex
 * functions); totals W_{s,k} - f_ext . u per part (reading R6) */
int oracle_quad_energy(int type, int64_t n_nodes, int64_t n_elems, const double* coords, const int32_t* conn,
                       int model, const double* mu, const double* lam, int n_samples, const double* u,
                       int n_parts, const int32_t* part_elem, const int32_t* part_node, const double* f_ext,
                       double* W_e, double* totals) {
    const int nv = quad_nv(type);
    double pts[18], w[9];
    const int nq = oracle_quad_rule(type, pts, w);
    double* W = W_e ? W_e : (double*)malloc(sizeof(double) * (size_t)n_elems * n_samples);
    if (!W) return OR_ERR_CAPACITY;
    int64_t first_bad = -1;
    for (int s = 0; s < n_samples; ++s) {
        const double* us = u + (int64_t)s * n_nodes * 2;
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < n_elems; ++e) {
            double We = 0.0;
            for (int q = 0; q < nq; ++q) {
                double g[8][2];
                const double det = quad_qp(type, coords, conn + e * nv, pts[2 * q], pts[2 * q + 1], g);
                if (quad_point(nv, model, g, w[q] * det, mu[e], lam[e], conn + e * nv, us, &We, NULL) != OR_OK) {
#pragma omp critical
                    { if (first_bad < 0 || e < first_bad) first_bad = e; }
                }
            }
            W[(int64_t)s * n_elems + e] = We;
        }
        for (int k = 0; k < n_parts; ++k) {
            double acc = 0.0;
            for (int64_t e = part_elem[k]; e < part_elem[k + 1]; ++e) acc += W[(int64_t)s * n_elems + e];
            if (f_ext) {
                double work = 0.0;
                for (int64_t n = part_node[k]; n < part_node[k + 1]; ++n)
                    for (int i = 0; i < 2; ++i) work += f_ext[n * 2 + i] * us[n * 2 + i];
                acc -= work;
            }
            totals[(int64_t)s * n_parts + k] = acc;
        }
    }
    if (!W_e) free(W);
    if (first_bad >= 0) { g_err_index = first_bad; return OR_ERR_INVERTED; }
    return OR_OK;
}

int oracle_quad_residual(int type, int64_t n_nodes, int64_t n_elems, const double* coords, const int32_t* conn,
                         int model, const double* mu, const double* lam, int n_samples, const double* u,
                         double* r) {
    const int nv = quad_nv(type), ne = 2 * nv;
    double pts[18], w[9];
    const int nq = oracle_quad_rule(type, pts, w);
    double* fe = (double*)malloc(sizeof(double) * (size_t)n_elems * ne);
    if (!fe) return OR_ERR_CAPACITY;
    int64_t first_bad = -1;
    for (int s = 0; s < n_samples; ++s) {
        const double* us = u + (int64_t)s * n_nodes * 2;
        double* rs = r + (int64_t)s * n_nodes * 2;
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < n_elems; ++e) {
            double* f = fe + e * ne;
            for (int k = 0; k < ne; ++k) f[k] = 0.0;
            for (int q = 0; q < nq; ++q) {
                double g[8][2];
                const double det = quad_qp(type, coords, conn + e * nv, pts[2 * q], pts[2 * q + 1], g);
                if (quad_point(nv, model, g, w[q] * det, mu[e], lam[e], conn + e * nv, us, NULL, f) != OR_OK) {
#pragma omp critical
                    { if (first_bad < 0 || e < first_bad) first_bad = e; }
                }
            }
        }
        for (int64_t k = 0; k < n_nodes * 2; ++k) rs[k] = 0.0;
        for (int64_t e = 0; e < n_elems; ++e)
            for (int a = 0; a < nv; ++a)
                for (int i = 0; i < 2; ++i) rs[(int64_t)conn[e * nv + a] * 2 + i] += fe[e * ne + 2 * a + i];
    }
    free(fe);
    if (first_bad >= 0) { g_err_index = first_bad; return OR_ERR_INVERTED; }
    return OR_OK;
}

int oracle_quad_tangent(int type, int64_t n_nodes, int64_t n_elems, const double* coords, const int32_t* conn,
                        int model, const double* mu, const double* lam, int n_samples, const double* u,
                        const double* v, const uint8_t* mask, double* Kv) {
    const int nv = quad_nv(type), ne = 2 * nv;
    double pts[18], w[9];
    const int nq = oracle_quad_rule(type, pts, w);
    double* fe = (double*)malloc(sizeof(double) * (size_t)n_elems * ne);
    if (!fe) return OR_ERR_CAPACITY;
    int64_t first_bad = -1;
    for (int s = 0; s < n_samples; ++s) {
        const double* vs = v + (int64_t)s * n_nodes * 2;
        const double* us = u ? u + (int64_t)s * n_nodes * 2 : NULL;
        double* out = Kv + (int64_t)s * n_nodes * 2;
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < n_elems; ++e) {
            const int32_t* c = conn + e * nv;
            double ve[16];
            for (int a = 0; a < nv; ++a)
                for (int i = 0; i < 2; ++i) {
                    const int64_t dof = (int64_t)c[a] * 2 + i;
                    ve[2 * a + i] = (mask && mask[dof]) ? 0.0 : vs[dof];
                }
            double* f = fe + e * ne;
            for (int k = 0; k < ne; ++k) f[k] = 0.0;
            for (int q = 0; q < nq; ++q) {
                double g[8][2];
                const double det = quad_qp(type, coords, c, pts[2 * q], pts[2 * q + 1], g);
                if (quad_point_tangent(nv, model, g, w[q] * det, mu[e], lam[e], c, us, ve, f) != OR_OK) {
#pragma omp critical
                    { if (first_bad < 0 || e < first_bad) first_bad = e; }
                }
            }
        }
        for (int64_t k = 0; k < n_nodes * 2; ++k) out[k] = 0.0;
        for (int64_t e = 0; e < n_elems; ++e)
            for (int a = 0; a < nv; ++a)
                for (int i = 0; i < 2; ++i) out[(int64_t)conn[e * nv + a] * 2 + i] += fe[e * ne + 2 * a + i];
        if (mask)
            for (int64_t k = 0; k < n_nodes * 2; ++k)
                if (mask[k]) out[k] = vs[k];
    }
    free(fe);
    if (first_bad >= 0) { g_err_index = first_bad; return OR_ERR_INVERTED; }
    return OR_OK;
}

struct quad_op {
    int type; int64_t n_nodes, n_elems; const double* coords; const int32_t* conn;
    int model; const double* mu; const double* lam; const double* u_state;
};
static int quad_apply(void* ctx, const double* v, const uint8_t* mask, double* out) {
    const struct quad_op* o = (const struct quad_op*)ctx;
    return oracle_quad_tangent(o->type, o->n_nodes, o->n_elems, o->coords, o->conn, o->model, o->mu, o->lam, 1,
                               o->u_state, v, mask, out);
}

int oracle_quad_cg(int type, int64_t n_nodes, int64_t n_elems, const double* coords, const int32_t* conn,
                   int model, const double* mu, const double* lam, const double* u_state, const double* f,
                   const uint8_t* mask, double* x, double tol, int32_t max_iter, double* history,
                   int32_t* iterations, double* rel_res0, double* rel_res_final, double* true_rel_res_final) {
    struct quad_op o = {type, n_nodes, n_elems, coords, conn, model, mu, lam, u_state};
    return cg_core(n_nodes * 2, quad_apply, &o, f, mask, x, tol, max_iter, history, iterations, rel_res0,
                   rel_res_final, true_rel_res_final);
}

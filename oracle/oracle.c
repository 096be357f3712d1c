/*
 * oracle.c -- plain, slow, obviously-correct CPU reference for the tcx hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2205_10091_b200/)
 * may include, link or call this file.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it.  It shares no code,
 * header, table or constant with the CUDA path: gate kinds are its own enum and
 * the Python wrapper (oracle/oracle.py) maps gate *names* to it.
 *
 * What it computes (each step cites the paper passage):
 *   psi(theta) = U_L(theta) ... U_1(theta) |0...0>           PAPER.md:391 (default
 *                all-zero input), :268-280 (gate-by-gate circuit, state()).
 *   E = Re sum_j alpha_j <psi|P_j|psi>                        PAPER.md:89-91 (Eq. 2),
 *                evaluated by the explicit loop of PAPER.md:818-829 (one
 *                expectation_ps per term; each P_j applied qubit by qubit).
 *   dE/dtheta  by the adjoint sweep (SURVEY §8 "Adjoint gradient"; PAPER.md:487-492
 *                defines the quantity as the exact derivative), and independently
 *                by the parameter-shift rule.
 * Precision: float64 complex throughout (C99 double complex), single threaded
 * except the optional OpenMP loop over independent theta rows.
 *
 * Conventions:
 *   qubit 0 = most significant bit: amplitude index r = sum_q b_q 2^{n-1-q}
 *           (PAPER.md:249, :278-280).
 *   R_P(a) = exp(-i a P / 2), a = coeff*theta[param] or coeff if param < 0
 *           (SPEC.md:221).
 *   2-qubit matrix on (q0,q1): row/col index 2*b_q0 + b_q1;
 *           CNOT control = q0.
 *   Pauli codes 0=I 1=X 2=Y 3=Z.
 */
#define _GNU_SOURCE
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

enum {
    OK_I = 0, OK_X, OK_Y, OK_Z, OK_H, OK_S, OK_SDG, OK_T, OK_TDG,
    OK_CNOT, OK_CZ, OK_SWAP,
    OK_RX, OK_RY, OK_RZ, OK_RXX, OK_RYY, OK_RZZ,
    OK_U1, OK_U2, OK_DEPOL, OK_RROT, OK_NKINDS
};

/* ---------------------------------------------------------------- matrices */
static void pauli2(int which, cplx m[4])
{   /* 1=X 2=Y 3=Z 0=I, textbook definitions */
    m[0] = m[1] = m[2] = m[3] = 0;
    if (which == 0) { m[0] = 1; m[3] = 1; }
    if (which == 1) { m[1] = 1; m[2] = 1; }
    if (which == 2) { m[1] = -I; m[2] = I; }
    if (which == 3) { m[0] = 1; m[3] = -1; }
}

static void kron22(const cplx a[4], const cplx b[4], cplx out[16])
{   /* (a (x) b)[(i*2+k),(j*2+l)] = a[i][j] b[k][l] */
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            for (int k = 0; k < 2; ++k)
                for (int l = 0; l < 2; ++l)
                    out[(i * 2 + k) * 4 + (j * 2 + l)] = a[i * 2 + j] * b[k * 2 + l];
}

static int arity(int kind)
{
    switch (kind) {
    case OK_CNOT: case OK_CZ: case OK_SWAP: case OK_RXX: case OK_RYY: case OK_RZZ: case OK_U2:
        return 2;
    default:
        return 1;
    }
}

static int is_rotation(int kind)
{
    return kind == OK_RX || kind == OK_RY || kind == OK_RZ ||
           kind == OK_RXX || kind == OK_RYY || kind == OK_RZZ || kind == OK_RROT;
}

/* The gate actually applied by gate g for this theta row: a random-axis rotation
 * (PAPER.md:1693-1704 unitary_kraus over [Rx, Ry, Rz], probabilities 1/3, external status)
 * becomes Rx / Ry / Rz by the row's status x = theta[s] (s = the payload's real part):
 * x < 1/3, x < 2/3, else. */
static int row_kind(int g, const int *kind, const int64_t *moff, const double *mats,
                    const double *theta)
{
    if (kind[g] != OK_RROT) return kind[g];
    const double x = theta[(int)mats[2 * moff[g]]];
    return x < 1.0 / 3.0 ? OK_RX : (x < 2.0 / 3.0 ? OK_RY : OK_RZ);
}

/* Pauli generator of a rotation gate: P with R_P(a) = exp(-i a P/2). */
static void generator(int kind, cplx *m /* 4 or 16 */)
{
    cplx p[4];
    switch (kind) {
    case OK_RX: pauli2(1, m); break;
    case OK_RY: pauli2(2, m); break;
    case OK_RZ: pauli2(3, m); break;
    case OK_RXX: pauli2(1, p); kron22(p, p, m); break;
    case OK_RYY: pauli2(2, p); kron22(p, p, m); break;
    case OK_RZZ: pauli2(3, p); kron22(p, p, m); break;
    }
}

/* Gate matrix (row-major).  Fixed gates: PAPER.md:343-360 (S = diag(1,i) at :355),
 * rotations exp(-i a P/2) = cos(a/2) I - i sin(a/2) P (P^2 = I), payloads as given. */
static void gate_matrix(int kind, double a, const double *payload, cplx *m)
{
    const double r2 = 1.0 / sqrt(2.0);
    int d = arity(kind) == 1 ? 2 : 4;
    memset(m, 0, sizeof(cplx) * d * d);
    switch (kind) {
    case OK_I: m[0] = 1; m[3] = 1; break;
    case OK_X: pauli2(1, m); break;
    case OK_Y: pauli2(2, m); break;
    case OK_Z: pauli2(3, m); break;
    case OK_H: m[0] = r2; m[1] = r2; m[2] = r2; m[3] = -r2; break;
    case OK_S: m[0] = 1; m[3] = I; break;
    case OK_SDG: m[0] = 1; m[3] = -I; break;
    case OK_T: m[0] = 1; m[3] = cexp(I * M_PI / 4); break;
    case OK_TDG: m[0] = 1; m[3] = cexp(-I * M_PI / 4); break;
    case OK_CNOT: m[0] = 1; m[5] = 1; m[11] = 1; m[14] = 1; break;
    case OK_CZ: m[0] = 1; m[5] = 1; m[10] = 1; m[15] = -1; break;
    case OK_SWAP: m[0] = 1; m[6] = 1; m[9] = 1; m[15] = 1; break;
    case OK_RX: case OK_RY: case OK_RZ: case OK_RXX: case OK_RYY: case OK_RZZ: {
        cplx g[16];
        generator(kind, g);
        for (int i = 0; i < d * d; ++i)
            m[i] = -I * sin(a / 2) * g[i];
        for (int i = 0; i < d; ++i)
            m[i * d + i] += cos(a / 2);
        break;
    }
    case OK_U1: case OK_U2:
        for (int i = 0; i < d * d; ++i)
            m[i] = payload[2 * i] + I * payload[2 * i + 1];
        break;
    case OK_DEPOL: {
        /* Monte Carlo trajectory of the depolarizing channel: [0,1) is
         * partitioned into intervals of lengths 1-px-py-pz, px, py, pz in the order of the
         * Kraus operators K0 = I, K1 = X, K2 = Y, K3 = Z; the status x = a picks the one
         * applied.  payload = (px, py, pz, 0). */
        const double px = payload[0], py = payload[1], pz = payload[2];
        int w = 0;
        if (a >= 1.0 - px - py - pz) w = 1;
        if (a >= 1.0 - py - pz) w = 2;
        if (a >= 1.0 - pz) w = 3;
        pauli2(w, m);
        break;
    }
    }
}

static void dagger(const cplx *m, int d, cplx *out)
{
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j)
            out[i * d + j] = conj(m[j * d + i]);
}

/* ----------------------------------------------------- gate application */
/* Apply a 2x2 matrix to qubit q: loop over every index with bit (n-1-q) clear. */
static void apply1(int n, cplx *psi, int q, const cplx m[4])
{
    const int64_t N = (int64_t)1 << n;
    const int64_t bit = (int64_t)1 << (n - 1 - q);
    for (int64_t r = 0; r < N; ++r) {
        if (r & bit) continue;
        cplx a = psi[r], b = psi[r | bit];
        psi[r] = m[0] * a + m[1] * b;
        psi[r | bit] = m[2] * a + m[3] * b;
    }
}

/* Apply a 4x4 matrix to (qa, qb); local index k = 2*b_qa + b_qb. */
static void apply2(int n, cplx *psi, int qa, int qb, const cplx m[16])
{
    const int64_t N = (int64_t)1 << n;
    const int64_t ba = (int64_t)1 << (n - 1 - qa);
    const int64_t bb = (int64_t)1 << (n - 1 - qb);
    for (int64_t r = 0; r < N; ++r) {
        if ((r & ba) || (r & bb)) continue;
        int64_t idx[4] = { r, r | bb, r | ba, r | ba | bb };
        cplx v[4], w[4];
        for (int k = 0; k < 4; ++k) v[k] = psi[idx[k]];
        for (int i = 0; i < 4; ++i) {
            w[i] = 0;
            for (int k = 0; k < 4; ++k) w[i] += m[i * 4 + k] * v[k];
        }
        for (int k = 0; k < 4; ++k) psi[idx[k]] = w[k];
    }
}

static void apply_matrix(int n, cplx *psi, int kind, int q0, int q1, const cplx *m)
{
    if (arity(kind) == 1) apply1(n, psi, q0, m);
    else apply2(n, psi, q0, q1, m);
}

static cplx inner(int64_t N, const cplx *a, const cplx *b)
{   /* <a|b> */
    cplx s = 0;
    for (int64_t r = 0; r < N; ++r) s += conj(a[r]) * b[r];
    return s;
}

/* ---------------------------------------------------------- validation */
/* returns 0 if valid, else 1 + index of the first offending gate */
int orc_validate(int n, int G, const int *kind, const int *q0, const int *q1,
                 const int *param, const int64_t *moff, int64_t nmat, int P)
{
    if (n < 1 || n > 30) return -1;
    for (int g = 0; g < G; ++g) {
        int k = kind[g];
        if (k < 0 || k >= OK_NKINDS) return 1 + g;
        if (q0[g] < 0 || q0[g] >= n) return 1 + g;
        if (arity(k) == 2 && (q1[g] < 0 || q1[g] >= n || q1[g] == q0[g])) return 1 + g;
        if (is_rotation(k) && (param[g] < -1 || param[g] >= P)) return 1 + g;
        if (k == OK_DEPOL && (param[g] < 0 || param[g] >= P || moff[g] < 0 || moff[g] + 2 > nmat))
            return 1 + g;
        if (k == OK_RROT && (moff[g] < 0 || moff[g] + 1 > nmat)) return 1 + g;
        if (k == OK_U1 || k == OK_U2) {
            int64_t need = (k == OK_U1 ? 4 : 16);
            if (moff[g] < 0 || moff[g] + need > nmat) return 1 + g;
        }
    }
    return 0;
}

static double angle_of(int g, const int *param, const double *coeff, const double *theta,
                       int shift_gate, double shift)
{
    double a = param[g] >= 0 ? coeff[g] * theta[param[g]] : coeff[g];
    if (g == shift_gate) a += shift;
    return a;
}

/* the argument gate_matrix takes: the angle, or for OK_DEPOL the row's status theta[param] */
static double gate_arg(int g, const int *kind, const int *param, const double *coeff,
                       const double *theta, int shift_gate, double shift)
{
    if (kind[g] == OK_DEPOL) return theta[param[g]];
    return angle_of(g, param, coeff, theta, shift_gate, shift);
}

/* ------------------------------------------------------------- state() */
/* psi = U_G ... U_1 |psi0>, psi0 = |0..0> when NULL (PAPER.md:391 default input) or
 * the caller's input state ("inputs" batched with the parameters,
 * SURVEY §8f f2); gate `shift_gate` gets its angle shifted by `shift` (used only by the
 * parameter-shift gradient).  out: 2^n interleaved (re, im). */
static void state_c(int n, int G, const int *kind, const int *q0, const int *q1,
                    const int *param, const double *coeff, const int64_t *moff,
                    const double *mats, const double *theta, int shift_gate, double shift,
                    cplx *psi, const cplx *psi0)
{
    const int64_t N = (int64_t)1 << n;
    if (psi0) {
        memcpy(psi, psi0, sizeof(cplx) * N);
    } else {
        for (int64_t r = 0; r < N; ++r) psi[r] = 0;
        psi[0] = 1;                               /* PAPER.md:391 default input */
    }
    for (int g = 0; g < G; ++g) {
        cplx m[16];
        double a = gate_arg(g, kind, param, coeff, theta, shift_gate, shift);
        const int k = row_kind(g, kind, moff, mats, theta);
        gate_matrix(k, a, moff[g] >= 0 ? mats + 2 * moff[g] : NULL, m);
        apply_matrix(n, psi, k, q0[g], q1[g], m);
    }
}

int orc_state(int n, int G, const int *kind, const int *q0, const int *q1,
              const int *param, const double *coeff, const int64_t *moff,
              const double *mats, const double *theta, double *out)
{
    state_c(n, G, kind, q0, q1, param, coeff, moff, mats, theta, -1, 0.0, (cplx *)out, NULL);
    return 0;
}

int orc_state_in(int n, int G, const int *kind, const int *q0, const int *q1,
                 const int *param, const double *coeff, const int64_t *moff,
                 const double *mats, const double *theta, const double *psi0, double *out)
{
    state_c(n, G, kind, q0, q1, param, coeff, moff, mats, theta, -1, 0.0, (cplx *)out,
            (const cplx *)psi0);
    return 0;
}

/* --------------------------------------------------- Pauli expectation */
/* P psi with P = sigma_{code[0]} (x) ... (x) sigma_{code[n-1]}: each single-qubit
 * Pauli applied in turn as a gate (PAPER.md:794-815 structures; :818-829 loop). */
static void pauli_apply(int n, const unsigned char *code, const cplx *psi, cplx *out)
{
    const int64_t N = (int64_t)1 << n;
    memcpy(out, psi, sizeof(cplx) * N);
    for (int q = 0; q < n; ++q) {
        if (code[q] == 0) continue;
        cplx m[4];
        pauli2(code[q], m);
        apply1(n, out, q, m);
    }
}

/* H psi = sum_j alpha_j P_j psi */
static void hamiltonian_apply(int n, int T, const unsigned char *codes, const double *w,
                              const cplx *psi, cplx *out, cplx *tmp)
{
    const int64_t N = (int64_t)1 << n;
    for (int64_t r = 0; r < N; ++r) out[r] = 0;
    for (int j = 0; j < T; ++j) {
        pauli_apply(n, codes + (int64_t)j * n, psi, tmp);
        for (int64_t r = 0; r < N; ++r) out[r] += w[j] * tmp[r];
    }
}

/* e[0] + i e[1] = sum_j alpha_j <psi|P_j|psi>  (the explicit loop
 * of :818-829).  Real part is E; the imaginary part must vanish. */
int orc_expect(int n, const double *state, int T, const unsigned char *codes,
               const double *w, double *e)
{
    const int64_t N = (int64_t)1 << n;
    const cplx *psi = (const cplx *)state;
    cplx *tmp = malloc(sizeof(cplx) * N);
    if (!tmp) return -2;
    cplx s = 0;
    for (int j = 0; j < T; ++j) {
        pauli_apply(n, codes + (int64_t)j * n, psi, tmp);
        s += w[j] * inner(N, psi, tmp);
    }
    free(tmp);
    e[0] = creal(s);
    e[1] = cimag(s);
    return 0;
}

static double energy(int n, int G, const int *kind, const int *q0, const int *q1,
                     const int *param, const double *coeff, const int64_t *moff,
                     const double *mats, const double *theta, int shift_gate, double shift,
                     int T, const unsigned char *codes, const double *w, cplx *psi)
{
    double e[2];
    state_c(n, G, kind, q0, q1, param, coeff, moff, mats, theta, shift_gate, shift, psi, NULL);
    orc_expect(n, (const double *)psi, T, codes, w, e);
    return e[0];
}

/* -------------------------------------------------------- adjoint sweep */
/* SURVEY §8 "Adjoint gradient": lambda_L = H psi_L; for g = L..1:
 *   if g has a parameter: grad[p] += coeff_g * Im <lambda|P_g|psi>   (both after g)
 *   psi <- U_g^dag psi; lambda <- U_g^dag lambda.
 * (d/da <psi|H|psi> with U = exp(-i a P/2) gives 2 Re <lambda|(-i/2) P|psi> = Im<lambda|P|psi>.)
 * E[0] = Re <psi|H|psi>, E[1] = Im (must be ~0). */
/* qim (optional, [P]): Im <psi|H|d psi / d theta_p>, the imaginary
 * part of the quantity whose real part is grad / 2: with psi = V U_g(a) W |psi0> and
 * dU_g/da = (-i/2) P_g U_g, <psi|H|d psi/da> = (-i/2) <lambda|P_g|psi> at gate g. */
static int value_grad_c(int n, int G, const int *kind, const int *q0, const int *q1,
                        const int *param, const double *coeff, const int64_t *moff,
                        const double *mats, int P, const double *theta,
                        int T, const unsigned char *codes, const double *w,
                        double *E, double *grad, const cplx *psi0, double *qim)
{
    const int64_t N = (int64_t)1 << n;
    cplx *psi = malloc(sizeof(cplx) * N), *lam = malloc(sizeof(cplx) * N);
    cplx *tmp = malloc(sizeof(cplx) * N);
    if (!psi || !lam || !tmp) { free(psi); free(lam); free(tmp); return -2; }
    state_c(n, G, kind, q0, q1, param, coeff, moff, mats, theta, -1, 0.0, psi, psi0);
    hamiltonian_apply(n, T, codes, w, psi, lam, tmp);
    cplx e = inner(N, psi, lam);
    E[0] = creal(e);
    E[1] = cimag(e);
    for (int p = 0; p < P; ++p) grad[p] = 0;
    if (qim)
        for (int p = 0; p < P; ++p) qim[p] = 0;
    for (int g = G - 1; g >= 0; --g) {
        const int k = row_kind(g, kind, moff, mats, theta);
        if (is_rotation(kind[g]) && param[g] >= 0) {
            cplx gen[16];
            generator(k, gen);
            memcpy(tmp, psi, sizeof(cplx) * N);
            apply_matrix(n, tmp, k, q0[g], q1[g], gen);
            const cplx z = inner(N, lam, tmp);       /* <lambda|P_g|psi> */
            grad[param[g]] += coeff[g] * cimag(z);  /* 2 Re((-i/2) z) */
            if (qim) qim[param[g]] += -0.5 * coeff[g] * creal(z);
        }
        cplx m[16], md[16];
        double a = gate_arg(g, kind, param, coeff, theta, -1, 0.0);
        gate_matrix(k, a, moff[g] >= 0 ? mats + 2 * moff[g] : NULL, m);
        dagger(m, arity(k) == 1 ? 2 : 4, md);
        apply_matrix(n, psi, k, q0[g], q1[g], md);
        apply_matrix(n, lam, k, q0[g], q1[g], md);
    }
    free(psi); free(lam); free(tmp);
    return 0;
}

int orc_value_grad(int n, int G, const int *kind, const int *q0, const int *q1,
                   const int *param, const double *coeff, const int64_t *moff,
                   const double *mats, int P, const double *theta,
                   int T, const unsigned char *codes, const double *w,
                   double *E, double *grad)
{
    return value_grad_c(n, G, kind, q0, q1, param, coeff, moff, mats, P, theta, T, codes, w,
                        E, grad, NULL, NULL);
}

int orc_value_qgrad(int n, int G, const int *kind, const int *q0, const int *q1,
                    const int *param, const double *coeff, const int64_t *moff,
                    const double *mats, int P, const double *theta,
                    int T, const unsigned char *codes, const double *w,
                    double *E, double *grad, double *qim)
{
    return value_grad_c(n, G, kind, q0, q1, param, coeff, moff, mats, P, theta, T, codes, w,
                        E, grad, NULL, qim);
}

/* ---------------------------------------------------- parameter shift */
/* For R_P(a), P^2 = I: E(a) = A + B cos a + C sin a, so dE/da = [E(a+pi/2) - E(a-pi/2)]/2
 * exactly; dE/dtheta_p = sum over gates g with param p of coeff_g * dE/da_g
 * (SURVEY §8c step 6).  Independent of the adjoint sweep above. */
int orc_param_shift(int n, int G, const int *kind, const int *q0, const int *q1,
                    const int *param, const double *coeff, const int64_t *moff,
                    const double *mats, int P, const double *theta,
                    int T, const unsigned char *codes, const double *w, double *grad)
{
    const int64_t N = (int64_t)1 << n;
    cplx *psi = malloc(sizeof(cplx) * N);
    if (!psi) return -2;
    for (int p = 0; p < P; ++p) grad[p] = 0;
    for (int g = 0; g < G; ++g) {
        if (!is_rotation(kind[g]) || param[g] < 0) continue;
        double ep = energy(n, G, kind, q0, q1, param, coeff, moff, mats, theta, g, M_PI / 2,
                           T, codes, w, psi);
        double em = energy(n, G, kind, q0, q1, param, coeff, moff, mats, theta, g, -M_PI / 2,
                           T, codes, w, psi);
        grad[param[g]] += coeff[g] * 0.5 * (ep - em);
    }
    free(psi);
    return 0;
}

/* ------------------------------------------------------ batched rows */
/* Rows are independent (PAPER.md:1121-1139 batched VQE; grad per row).
 * nthreads > 1 runs rows in parallel with OpenMP (used only for the reported CPU
 * baseline); the arithmetic per row is identical. */
/* psi0: NULL (all rows start from |0..0>) or [B][2^n] interleaved input states */
static int value_grad_batch_c(int n, int G, const int *kind, const int *q0, const int *q1,
                              const int *param, const double *coeff, const int64_t *moff,
                              const double *mats, int P, int B, const double *theta,
                              int T, const unsigned char *codes, const double *w,
                              double *E, double *grad, int nthreads, const double *psi0)
{
    int err = 0;
    const int64_t N = (int64_t)1 << n;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1) reduction(|:err)
#endif
    for (int b = 0; b < B; ++b)
        err |= value_grad_c(n, G, kind, q0, q1, param, coeff, moff, mats, P,
                            theta + (int64_t)b * P, T, codes, w, E + 2 * b,
                            grad + (int64_t)b * P,
                            psi0 ? (const cplx *)(psi0 + 2 * N * b) : NULL, NULL) != 0;
    (void)nthreads;
    return err ? -2 : 0;
}

int orc_value_grad_batch(int n, int G, const int *kind, const int *q0, const int *q1,
                         const int *param, const double *coeff, const int64_t *moff,
                         const double *mats, int P, int B, const double *theta,
                         int T, const unsigned char *codes, const double *w,
                         double *E /* [B][2] */, double *grad /* [B][P] */, int nthreads)
{
    return value_grad_batch_c(n, G, kind, q0, q1, param, coeff, moff, mats, P, B, theta, T,
                              codes, w, E, grad, nthreads, NULL);
}

int orc_value_grad_batch_in(int n, int G, const int *kind, const int *q0, const int *q1,
                            const int *param, const double *coeff, const int64_t *moff,
                            const double *mats, int P, int B, const double *theta,
                            int T, const unsigned char *codes, const double *w,
                            double *E, double *grad, int nthreads, const double *psi0)
{
    return value_grad_batch_c(n, G, kind, q0, q1, param, coeff, moff, mats, P, B, theta, T,
                              codes, w, E, grad, nthreads, psi0);
}

int orc_expect_batch(int n, int G, const int *kind, const int *q0, const int *q1,
                     const int *param, const double *coeff, const int64_t *moff,
                     const double *mats, int P, int B, const double *theta,
                     int T, const unsigned char *codes, const double *w,
                     double *E /* [B][2] */, int nthreads)
{
    int err = 0;
    const int64_t N = (int64_t)1 << n;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1) reduction(|:err)
#endif
    for (int b = 0; b < B; ++b) {
        cplx *psi = malloc(sizeof(cplx) * N);
        if (!psi) { err |= 1; continue; }
        state_c(n, G, kind, q0, q1, param, coeff, moff, mats, theta + (int64_t)b * P,
                -1, 0.0, psi, NULL);
        err |= orc_expect(n, (const double *)psi, T, codes, w, E + 2 * b) != 0;
        free(psi);
    }
    (void)nthreads;
    return err ? -2 : 0;
}

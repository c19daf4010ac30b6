/*
 * lamb_oracle.c — CPU ORACLE for the MegaScale LAMB step.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this.  It shares no code, header, table or constant generator with the
 * CUDA path in paper_2402_15627_b200/ (DESIGN.md §3).  Plain loops, IEEE double, no
 * -ffast-math, no blocking or fusion beyond what the definitions state.
 *
 * What it follows:
 *  - LAMB: PAPER.md §3.1 P:288-293 ("The LAMB optimizer~\cite{You2020Large}") — the paper
 *    prints no update rule, so the rule is the cited Algorithm 2 of You et al. (ICLR 2020)
 *    as read in DESIGN.md Z1-Z9, Z14:
 *        m <- b1 m + (1-b1) g ;  v <- b2 v + (1-b2) g^2
 *        mhat = m/(1-b1^t) ; vhat = v/(1-b2^t)          (bias correction, Z5)
 *        r = mhat / (sqrt(vhat) + eps)                   (eps outside the sqrt, Z4)
 *        u = r + lambda w                                (decoupled decay inside, Z1/Z7)
 *        ratio = adapt ? (|w|>0 && |u|>0 ? |w|/|u| : 1) : 1   (phi = id, Z3; fallback Z9)
 *        w <- w - lr * ratio * u
 *    one "layer" = one parameter tensor, norms over its numel elements (Z2).
 *  - ZeRO-2 DP semantics, §2: reduce-scatter + all-gather == all-reduce
 *    of the gradients followed by a replicated update; so the oracle reduces
 *    g = grad_scale * sum_j G_j (Z10/Z11) and updates unsharded tensors.
 *  - Synthetic inputs: Philox4x32-10 (Salmon et al., SC'11, Random123 definition) keyed as
 *    in DESIGN.md "Input recipe".
 *
 * Pins (tests/test_oracle_*.py): Random123 known-answer vectors; closed forms H1/H1b/H2/H3/
 * H4/H5; torch.optim.AdamW (float64) for adapt=0 (H6); ||dw|| = lr ||w|| (H7); shard-count
 * invariance (H8); numpy.linalg.norm (H9).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------- Philox4x32-10 (Salmon et al. 2011, Random123) ---------------- */
/* Multipliers and Weyl key increments as defined by Random123 philox.h. */
#define ORC_PHILOX_M0 0xD2511F53u
#define ORC_PHILOX_M1 0xCD9E8D57u
#define ORC_PHILOX_W0 0x9E3779B9u
#define ORC_PHILOX_W1 0xBB67AE85u

void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += ORC_PHILOX_W0; k1 += ORC_PHILOX_W1; }
        uint64_t p0 = (uint64_t)ORC_PHILOX_M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)ORC_PHILOX_M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* One 32-bit word of the input stream for element e of tensor `tensor_id`.
 * key = (seed lo, seed hi ^ stream<<24 ^ rank_term); ctr = (q lo, q hi, tensor, step), q=e/4;
 * element e uses word e mod 4. */
uint32_t orc_gen_word(uint64_t seed, uint32_t stream, uint32_t rank_term, uint32_t tensor_id,
                      uint32_t step, int64_t e) {
    uint64_t q = (uint64_t)e / 4u;
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu),
                       (uint32_t)(seed >> 32) ^ (stream << 24) ^ rank_term};
    uint32_t ctr[4] = {(uint32_t)(q & 0xFFFFFFFFu), (uint32_t)(q >> 32), tensor_id, step};
    uint32_t out[4];
    orc_philox4x32_10(ctr, key, out);
    return out[(uint64_t)e % 4u];
}

/* fp32 master weights: init 0 = uniform (int(x>>8) - 2^23) * 2^-23 * 2^-5, 1 = 1.0, 2 = 0.0 */
void orc_gen_weights(uint64_t seed, uint32_t tensor_id, int32_t init, int64_t numel, double* out) {
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < numel; ++e) {
        if (init == 1) { out[e] = 1.0; continue; }
        if (init == 2) { out[e] = 0.0; continue; }
        uint32_t x = orc_gen_word(seed, 1u, 0u, tensor_id, 0u, e);
        int64_t k = (int64_t)(x >> 8) - 8388608;          /* in [-2^23, 2^23) */
        out[e] = ldexp((double)k, -28);                  /* * 2^-23 * 2^-5 */
    }
}

/* bf16-representable gradients: 0 w.p. 1/16; else sign = bit 4,
 * value = +-(1 + mant/128) * 2^(gexp - ((x>>5)&3)), mant = (x>>7)&0x7F. */
void orc_gen_grads(uint64_t seed, uint32_t rank_term, uint32_t tensor_id, uint32_t step,
                   int32_t gexp, int64_t numel, double* out) {
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < numel; ++e) {
        uint32_t x = orc_gen_word(seed, 2u, rank_term, tensor_id, step, e);
        if ((x & 0xFu) == 0u) { out[e] = 0.0; continue; }
        int sign = (int)((x >> 4) & 1u);
        int ex = gexp - (int)((x >> 5) & 3u);
        int mant = (int)((x >> 7) & 0x7Fu);
        double mag = ldexp(1.0 + (double)mant / 128.0, ex);
        out[e] = sign ? -mag : mag;
    }
}

/* ---------------- LAMB, one parameter tensor ("layer", Z2) ---------------- */

/* Moments and the unscaled update u (You et al. Alg. 2 lines: m_t, v_t, bias-corrected
 * m_hat / v_hat, r_t = m_hat/(sqrt(v_hat)+eps), u = r_t + lambda x_t). */
void orc_moments_and_update(int64_t n, const double* w, double* m, double* v, const double* g,
                            double beta1, double beta2, double eps, double weight_decay,
                            int32_t bias_correction, int64_t t, double* u) {
    double bc1 = bias_correction ? 1.0 - pow(beta1, (double)t) : 1.0;
    double bc2 = bias_correction ? 1.0 - pow(beta2, (double)t) : 1.0;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        m[i] = beta1 * m[i] + (1.0 - beta1) * g[i];
        v[i] = beta2 * v[i] + (1.0 - beta2) * g[i] * g[i];
        double mhat = m[i] / bc1;
        double vhat = v[i] / bc2;
        double r = mhat / (sqrt(vhat) + eps);
        u[i] = r + weight_decay * w[i];
    }
}

/* sum of squares, one sequential loop (the plain definition of ||x||^2) */
double orc_sumsq(int64_t n, const double* x) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += x[i] * x[i];
    return s;
}

/* trust ratio, phi = identity (Z3), zero-norm fallback 1 (Z9); adapt=0 gives AdamW (Z8) */
double orc_trust_ratio(double w_norm, double u_norm, int32_t adapt) {
    if (!adapt) return 1.0;
    if (w_norm > 0.0 && u_norm > 0.0) return w_norm / u_norm;
    return 1.0;
}

/* w <- w - lr * ratio * u */
void orc_apply(int64_t n, double* w, const double* u, double lr, double ratio) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) w[i] = w[i] - lr * ratio * u[i];
}

/* One full LAMB step of one tensor; u is caller scratch of n doubles.
 * out3 = {||w_t||, ||u_t||, ratio} (w norm of the PRE-update weights). */
void orc_lamb_tensor_step(int64_t n, double* w, double* m, double* v, const double* g, double* u,
                          double lr, double beta1, double beta2, double eps, double weight_decay,
                          int32_t adapt, int32_t bias_correction, int64_t t, double* out3) {
    orc_moments_and_update(n, w, m, v, g, beta1, beta2, eps, weight_decay, bias_correction, t, u);
    double w_norm = sqrt(orc_sumsq(n, w));
    double u_norm = sqrt(orc_sumsq(n, u));
    double ratio = orc_trust_ratio(w_norm, u_norm, adapt);
    orc_apply(n, w, u, lr, ratio);
    out3[0] = w_norm; out3[1] = u_norm; out3[2] = ratio;
}

/* g = grad_scale * sum_{j=0..D-1} G_j (ZeRO-2 reduce, Z10/Z11), fixed order j = 0..D-1. */
void orc_reduce(int64_t n, int32_t D, const double* const* G, double grad_scale, double* g) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int32_t j = 0; j < D; ++j) s += G[j][i];
        g[i] = grad_scale * s;
    }
}

uint16_t orc_bf16_rne(double x);

/* The two bf16 numbers that bracket x (reading Z23, NVLS mode: the NVSwitch returns ONE of them
 * for the sum of the D ranks' bf16 gradients — a faithful, stochastically rounded bf16 sum;
 * measured, Z23).  lo = the largest bf16 <= x, hi = the smallest bf16 >= x (equal when x
 * is a bf16 number).  x must be finite and exactly representable in fp32 (the exact sum of
 * bf16 gradients under the input generator, H10).  Pure bit arithmetic on the fp32 pattern:
 * truncating the low 16 bits moves toward zero. */
void orc_bf16_neighbors(int64_t n, const double* x, double* lo, double* hi) {
    for (int64_t i = 0; i < n; ++i) {
        float f = (float)x[i];
        uint32_t b, t;
        memcpy(&b, &f, 4);
        t = b & 0xFFFF0000u;                       /* toward zero */
        float tz, away;
        memcpy(&tz, &t, 4);
        if (t == b) { lo[i] = hi[i] = (double)f; continue; }
        t += 0x10000u;                             /* next bf16 away from zero (same sign) */
        memcpy(&away, &t, 4);
        if (f > 0) { lo[i] = (double)tz; hi[i] = (double)away; }
        else { lo[i] = (double)away; hi[i] = (double)tz; }
    }
}

/* fp32 -> bf16 round-to-nearest-even of a double first rounded to float (Z15). */
uint16_t orc_bf16_rne(double x) {
    float f = (float)x;
    uint32_t b;
    memcpy(&b, &f, 4);
    if ((b & 0x7F800000u) == 0x7F800000u && (b & 0x7FFFFFu)) return (uint16_t)((b >> 16) | 0x40u);
    uint32_t lsb = (b >> 16) & 1u;
    b += 0x7FFFu + lsb;
    return (uint16_t)(b >> 16);
}

int32_t orc_num_threads(void) {
#ifdef _OPENMP
    return (int32_t)omp_get_max_threads();
#else
    return 1;
#endif
}

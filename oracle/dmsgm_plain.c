/*
 * dmsgm_plain.c -- TEST INFRASTRUCTURE ONLY (see dmsgm_oracle.h).
 *
 * Oracle form 1, "plain": one grid-block Dual-Mode SGM step written as SURVEY.md
 * §8(c)'s literal definition, with no evaluation-order choices beyond what that
 * definition writes:
 *   S1  fp64 projection of the block centre through H (R2-R5):
 *         w = (h6 X + h7 Y) + h8,  x' = ((h0 X + h1 Y) + h2) / w,  y' likewise;
 *   S2  every mixed sum divided by sum W (R6):
 *         mu~ = (sum_k W_k mu_k) / sum W,
 *         var~ = (sum_k W_k (var_k + (mu~ - mu_k)^2)) / sum W,
 *         age~ = min((sum_k W_k age_k) / sum W, cap);
 *   S3  age~ * (float) exp(-(double) lambda * (double)(var~ - theta_v))  (libm exp, R7);
 *   S6  Eqs. 3/5 in the incremental form of R10 with IEEE division:
 *         mu = mu~ + (M - mu~) / (age~ + 1),  var = var~ + (V - var~) / (age~ + 1).
 * Every + - * / is one IEEE round-to-nearest operation in the order written (built with
 * -ffp-contract=off; no fma anywhere).  Form 0 (dmsgm_oracle.c) evaluates the same
 * mathematics in the order the CUDA kernel uses; tests/test_oracle_forms.py pins form 0
 * against this file over whole synthetic sequences.
 *
 * The decisions of the step (match, reset, swap, exposure, mask) and readings R1, R7-R9,
 * R11-R16, R19-R29 are identical in both forms; only the arithmetic above differs.
 */
#include <math.h>

#include "oracle_ctx.h"

/* S1: source blocks and overlap weights of block (bi, bj).  Returns 1 if exposed (R5). */
static int plain_project(int Wb, int Hb, int N, const double* h, int bi, int bj, int kx[4], int ky[4],
                         float Wt[4], float* sumW) {
    double X = (double)N * bi + (double)N / 2.0;      /* block centre, R2 */
    double Y = (double)N * bj + (double)N / 2.0;
    double w = (h[6] * X + h[7] * Y) + h[8];
    if (!(w > 0.0)) return 1;                          /* R5: behind the camera */
    double xp = ((h[0] * X + h[1] * Y) + h[2]) / w;    /* R3: frame t -> frame t-1 */
    double yp = ((h[3] * X + h[4] * Y) + h[5]) / w;
    double u = xp / N, v = yp / N;                     /* source block-grid coordinates */
    if (!(u > -2.0 && u < Wb + 2.0 && v > -2.0 && v < Hb + 2.0)) return 1;   /* far out */
    double ku = floor(u), kv = floor(v);
    double du = u - (ku + 0.5), dv = v - (kv + 0.5);
    int su = du > 0.0 ? 1 : -1, sv = dv > 0.0 ? 1 : -1;
    float a = (float)fabs(du), b = (float)fabs(dv);
    Wt[0] = (1.0f - a) * (1.0f - b);                   /* self, H, V, HV (R4) */
    Wt[1] = a * (1.0f - b);
    Wt[2] = (1.0f - a) * b;
    Wt[3] = a * b;
    kx[0] = (int)ku;      ky[0] = (int)kv;
    kx[1] = (int)ku + su; ky[1] = (int)kv;
    kx[2] = (int)ku;      ky[2] = (int)kv + sv;
    kx[3] = (int)ku + su; ky[3] = (int)kv + sv;
    for (int k = 0; k < 4; ++k)
        if (kx[k] < 0 || kx[k] >= Wb || ky[k] < 0 || ky[k] >= Hb) Wt[k] = 0.0f;   /* R5 */
    *sumW = ((Wt[0] + Wt[1]) + Wt[2]) + Wt[3];
    return *sumW == 0.0f;
}

/* S2 + S3 for one model (A with A, C with C), R6 / R7. */
static sgm plain_mix(const dmsgm_oracle_ctx* c, const float* prev, int pm, const int kx[4], const int ky[4],
                     const float Wt[4], float sumW) {
    const size_t pe = oracle_plane_elems(c);
    float mu_k[4] = {0, 0, 0, 0}, var_k[4] = {0, 0, 0, 0}, age_k[4] = {0, 0, 0, 0};
    for (int k = 0; k < 4; ++k) {
        if (Wt[k] == 0.0f) continue;                   /* dropped source: contributes nothing */
        size_t idx = (size_t)ky[k] * (size_t)c->Wb + (size_t)kx[k];
        mu_k[k] = prev[(size_t)pm * pe + idx];
        var_k[k] = prev[(size_t)(pm + 1) * pe + idx];
        age_k[k] = prev[(size_t)(pm + 2) * pe + idx];
    }
    sgm m;
    m.mu = (((Wt[0] * mu_k[0] + Wt[1] * mu_k[1]) + Wt[2] * mu_k[2]) + Wt[3] * mu_k[3]) / sumW;
    float s[4];
    for (int k = 0; k < 4; ++k) {
        float d = m.mu - mu_k[k];
        s[k] = var_k[k] + d * d;
    }
    m.var = (((Wt[0] * s[0] + Wt[1] * s[1]) + Wt[2] * s[2]) + Wt[3] * s[3]) / sumW;
    float age = (((Wt[0] * age_k[0] + Wt[1] * age_k[1]) + Wt[2] * age_k[2]) + Wt[3] * age_k[3]) / sumW;
    m.age = age < c->p.age_cap ? age : c->p.age_cap;
    if (c->p.decay_lambda > 0.0f && m.var > c->p.decay_var_thresh)
        m.age = m.age * (float)exp(-(double)c->p.decay_lambda * (double)(m.var - c->p.decay_var_thresh));
    return m;
}

/* Eq. 6 over the block with the updated mean (App. E): the literal pixel loop. */
static float plain_V(float mu, const uint8_t* frame, size_t pitch, int x0, int y0, int N) {
    float V = -1.0f;
    for (int y = 0; y < N; ++y)
        for (int x = 0; x < N; ++x) {
            float e = mu - (float)frame[(size_t)(y0 + y) * pitch + (size_t)(x0 + x)];
            if (e * e > V) V = e * e;
        }
    return V;
}

/* Eqs. 3, 5, 7 (R10, R22), or the App. E rule (R27) when update_rule == 1. */
static sgm plain_update(const dmsgm_oracle_ctx* c, sgm t, float M, const uint8_t* frame, size_t pitch, int x0,
                        int y0) {
    sgm r;
    float den = t.age + 1.0f;
    if (c->p.update_rule == 0) {
        r.mu = t.mu + (M - t.mu) / den;
        float V = plain_V(r.mu, frame, pitch, x0, y0, c->N);
        r.var = t.var + (V - t.var) / den;
    } else {
        float alpha = 1.0f / (t.age > 1.0f ? t.age : 1.0f);     /* App. E */
        r.mu = (1.0f - alpha) * t.mu + alpha * M;
        float V = plain_V(r.mu, frame, pitch, x0, y0, c->N);
        r.var = (1.0f - alpha) * t.var + alpha * V;
    }
    r.age = den < c->p.age_cap ? den : c->p.age_cap;            /* Eq. 7, cap 30 */
    return r;
}

int dmsgm_plain_step_stream(dmsgm_oracle_ctx* c, int s, const uint8_t* frame, size_t fpitch, const double* h,
                            uint8_t* mask, size_t mpitch) {
    const int N = c->N, Wb = c->Wb, Hb = c->Hb;
    const size_t pe = oracle_plane_elems(c);
    const float* prev = oracle_stream_state(c, c->cur, s);
    float* next = oracle_stream_state(c, c->cur ^ 1, s);
    for (int bj = 0; bj < Hb; ++bj) {
        for (int bi = 0; bi < Wb; ++bi) {
            const int x0 = bi * N, y0 = bj * N;
            long sum = 0;                                            /* S4, Eq. 4 */
            for (int y = 0; y < N; ++y)
                for (int x = 0; x < N; ++x) sum += frame[(size_t)(y0 + y) * fpitch + (size_t)(x0 + x)];
            const float M = (float)sum / (float)(N * N);
            const sgm reset = {M, c->p.var_init, 1.0f};
            sgm A = reset, C = reset;                                /* S0 (R8) unless live */
            int kx[4], ky[4];
            float Wt[4], sumW;
            const int live = c->initialised[s] && !plain_project(Wb, Hb, N, h, bi, bj, kx, ky, Wt, &sumW);
            if (!live && c->dump) oracle_dump_tilde(c, s, bj, bi, reset, reset, M, 0);   /* test probe only */
            if (live) {
                sgm At = plain_mix(c, prev, P_MU_A, kx, ky, Wt, sumW);   /* S1-S3 */
                sgm Ct = plain_mix(c, prev, P_MU_C, kx, ky, Wt, sumW);
                if (c->dump) oracle_dump_tilde(c, s, bj, bi, At, Ct, M, 1);
                float dA = M - At.mu, dC = M - Ct.mu;                /* S5, Eqs. 8-9 */
                int matchA = dA * dA < c->p.theta_s * (At.var > c->p.var_floor_match ? At.var : c->p.var_floor_match);
                int matchC = !matchA &&
                             dC * dC < c->p.theta_s * (Ct.var > c->p.var_floor_match ? Ct.var : c->p.var_floor_match);
                if (matchA) {                                        /* S6 */
                    A = plain_update(c, At, M, frame, fpitch, x0, y0);
                    C = Ct;
                } else if (matchC) {
                    A = At;
                    C = plain_update(c, Ct, M, frame, fpitch, x0, y0);
                } else {
                    A = At;
                    C = reset;
                }
                if (C.age > A.age) {                                 /* S7, Eq. 10 */
                    A = C;
                    C = reset;
                }
            }
            for (int y = 0; y < N; ++y)                              /* S8, App. E */
                for (int x = 0; x < N; ++x) {
                    float I = (float)frame[(size_t)(y0 + y) * fpitch + (size_t)(x0 + x)];
                    float floor_of = c->p.classify_rule == 0 ? A.var : I;
                    float T = c->p.theta_d * (floor_of > c->p.var_floor_classify ? floor_of : c->p.var_floor_classify);
                    float d = I - A.mu;
                    mask[(size_t)(y0 + y) * mpitch + (size_t)(x0 + x)] = (d * d > T) ? 255 : 0;
                }
            size_t idx = (size_t)bj * (size_t)Wb + (size_t)bi;       /* S9 */
            next[P_MU_A * pe + idx] = A.mu;
            next[P_VAR_A * pe + idx] = A.var;
            next[P_AGE_A * pe + idx] = A.age;
            next[P_MU_C * pe + idx] = C.mu;
            next[P_VAR_C * pe + idx] = C.var;
            next[P_AGE_C * pe + idx] = C.age;
        }
    }
    return 0;
}

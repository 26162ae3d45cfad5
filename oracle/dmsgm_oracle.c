/*
 * dmsgm_oracle.c -- TEST INFRASTRUCTURE ONLY (see dmsgm_oracle.h).
 *
 * Plain single-threaded CPU oracle of one grid-block Dual-Mode SGM step,
 * written step by step in the paper's order and notation:
 *
 *   tilde models  (mu~, sigma~, alpha~) = previous models after motion
 *                  compensation (§2.2), computed here as Yi et al.'s
 *                  "mixture between grid blocks based on this homography
 *                  matrix" (§2.4) -- readings R2-R7 -- plus age decay (R7);
 *   M_i           block mean, Eq. 4, general |G_i| = N*N;
 *   match test    Eqs. 8-9, App. E P:605/P:620 floors;
 *   update        Eqs. 3, 5, 6, 7 for the matched model;
 *   reset         candidate reset (App. E);
 *   swap          Eq. 10 (App. E);
 *   mask          App. E P:655-663 with the variance reading R14.
 *
 * Arithmetic: fp32 throughout (north_star: "fp32 means/variances"); the
 * projection is in displacement form (R17), the decay exp a fixed fp32
 * sequence (R18); fp64 only converts the homography.  Built
 * with -O2 -ffp-contract=off -fno-fast-math: every + - * / below is one IEEE
 * round-to-nearest operation evaluated in the order written; fused
 * multiply-adds appear only where written as fma()/fmaf() (correctly rounded,
 * C99), never by contraction.  x*x is used, never pow.
 *
 * Layout: state [S][6][Hb][Wb] fp32, planes mu_A var_A age_A mu_C var_C age_C.
 */
#include "dmsgm_oracle.h"
#include "oracle_ctx.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static size_t plane_elems(const dmsgm_oracle_ctx* c) { return oracle_plane_elems(c); }

static float* stream_state(const dmsgm_oracle_ctx* c, int buf, int s) { return oracle_stream_state(c, buf, s); }

/* ------------------------------------------------------------------------
 * S1: project the block centre through H and find the up-to-4 source blocks
 * with their overlap (bilinear) weights.  Readings R2 (coordinates), R3 (H maps
 * frame t -> frame t-1), R4 (axis-aligned N x N footprint centred at H(c)),
 * R5 (out-of-range sources dropped; exposed block if w <= 0, if the displacement
 * is not finite / beyond 2^20 blocks, or if no in-range source has weight), R17
 * (displacement form in fp32: with g = H - I and e = w - 1,
 *   (x' - X) w = g0 X + g1 Y + g2 - X e,   (y' - Y) w = g3 X + g4 Y + g5 - Y e,
 * so the block-unit displacement (ex, ey) = ((x'-X)/N, (y'-Y)/N) keeps ~1e-7
 * accuracy for the near-identity homographies of a moving camera).
 * Returns 1 if exposed.
 * ---------------------------------------------------------------------- */
static int project_block(int Wb, int Hb, int N, const double* h, int bi, int bj,
                         int kx[4], int ky[4], float Wt[4], float* sumW, int* clipped) {
    const float g0 = (float)(h[0] - 1.0), g1 = (float)h[1], g2 = (float)h[2];
    const float g3 = (float)h[3], g4 = (float)(h[4] - 1.0), g5 = (float)h[5];
    const float g6 = (float)h[6], g7 = (float)h[7], g8 = (float)(h[8] - 1.0);
    float X = (float)(N * bi) + (float)N / 2.0f; /* block centre, R2 (exact in fp32) */
    float Y = (float)(N * bj) + (float)N / 2.0f;
    float e = fmaf(g6, X, fmaf(g7, Y, g8));      /* w - 1 */
    float w = 1.0f + e;
    if (!(w > 0x1p-100f && w < 0x1p100f)) return 1;   /* R5: w <= 0 or a degenerate projective scale */
    float px = fmaf(-X, e, fmaf(g0, X, fmaf(g1, Y, g2)));
    float py = fmaf(-Y, e, fmaf(g3, X, fmaf(g4, Y, g5)));
    float rw = 1.0f / w;
    float ex = (px * rw) / (float)N;             /* displacement of the centre in blocks */
    float ey = (py * rw) / (float)N;
    if (!(fabsf(ex) < 1048576.0f && fabsf(ey) < 1048576.0f)) return 1;
    /* source block-grid coordinate u = bi + 1/2 + ex: block k covers [k, k+1) */
    float tx = 0.5f + ex, ty = 0.5f + ey;
    float fx = floorf(tx), fy = floorf(ty);
    float du = (tx - fx) - 0.5f;                 /* offset of the footprint centre from the source block centre */
    float dv = (ty - fy) - 0.5f;
    int ku = bi + (int)fx, kv = bj + (int)fy;
    int su = du > 0.0f ? 1 : -1;
    int sv = dv > 0.0f ? 1 : -1;
    float a = fabsf(du);
    float b = fabsf(dv);
    float one_a = 1.0f - a;
    float one_b = 1.0f - b;
    /* overlap areas of the unit footprint with the 4 cells, order self, H, V, HV */
    Wt[0] = one_a * one_b;
    Wt[1] = a * one_b;
    Wt[2] = one_a * b;
    Wt[3] = a * b;
    kx[0] = ku;       ky[0] = kv;
    kx[1] = ku + su;  ky[1] = kv;
    kx[2] = ku;       ky[2] = kv + sv;
    kx[3] = ku + su;  ky[3] = kv + sv;
    *clipped = 0;
    for (int k = 0; k < 4; ++k)
        if (kx[k] < 0 || kx[k] >= Wb || ky[k] < 0 || ky[k] >= Hb) {
            if (Wt[k] > 0.0f) *clipped = 1;   /* part of the footprint lies outside the grid */
            Wt[k] = 0.0f;
        }
    float sw = Wt[0] + Wt[1];
    sw = sw + Wt[2];
    sw = sw + Wt[3];
    *sumW = sw;
    if (sw == 0.0f) return 1;
    return 0;
}

/* ------------------------------------------------------------------------
 * R18: the decay factor exp(-lambda * d), d = var~ - theta_v >= 0, in fp32 by one fixed
 * sequence of IEEE operations (so that any two IEEE machines agree bitwise), accurate
 * to about one fp32 ulp of the plain form's (float) exp(-(double) lambda * (double) d):
 *   x = lambda * d exactly as xh + xl (xh = fl(lambda d), xl = fma(lambda, d, -xh));
 *   n = rint(xh * log2 e);  r = fma(-n, L1, xh) + xl;  r = fma(-n, L2, r)
 *     (L1 + L2 = ln 2; L1 has 16 significant bits, so n*L1 is exact for n < 128);
 *   p = sum_{k=0..7} (-r)^k / k!  by Horner with fma from k = 7 down;  exp(-x) = p * 2^-n.
 * xh >= 86 returns 0 (exp(-86) is within 3 binades of FLT_MIN).
 * ---------------------------------------------------------------------- */
static float decay_factor(float lambda, float d) {
    const float xh = lambda * d;
    const float xl = fmaf(lambda, d, -xh);
    if (!(xh < 86.0f)) return 0.0f;
    const float n = rintf(xh * 1.44269502f);
    float r = fmaf(-n, 0.693145751953125f, xh) + xl;
    r = fmaf(-n, 1.42860677e-06f, r);
    float p = -1.98412701e-04f;            /* -1/7! */
    p = fmaf(p, r, 1.38888892e-03f);       /*  1/6! */
    p = fmaf(p, r, -8.33333377e-03f);      /* -1/5! */
    p = fmaf(p, r, 4.16666679e-02f);       /*  1/4! */
    p = fmaf(p, r, -1.66666672e-01f);      /* -1/3! */
    p = fmaf(p, r, 0.5f);                  /*  1/2! */
    p = fmaf(p, r, -1.0f);                 /* -1/1! */
    p = fmaf(p, r, 1.0f);                  /*  1/0! */
    return p * ldexpf(1.0f, -(int)n);
}

/* ------------------------------------------------------------------------
 * S2: mix one model (A with A, C with C) over the sources, reading R6:
 *   w_k = W_k                               (overlap areas of the unit footprint), or
 *   w_k = W_k / sum W  if part of the footprint fell outside the grid (renormalised)
 *   mu~  = sum_k w_k mu_k
 *   var~ = sum_k w_k (var_k + (mu~ - mu_k)^2)   (mixture second moment about mu~)
 *   age~ = min(sum_k w_k age_k, cap)
 * Sums run over in-range sources in the order self, H, V, HV, accumulated with
 * fused multiply-adds acc = fma(w_k, x_k, acc) from acc = 0 (R17).
 * S3: age decay (R7): if lambda > 0 and var~ > theta_v,
 *   age~ <- age~ * exp(-lambda (var~ - theta_v))   with exp as in decay_factor (R18).
 * ---------------------------------------------------------------------- */
static sgm mix_model(const dmsgm_oracle_ctx* c, const float* prev, int pm, const int kx[4],
                     const int ky[4], const float wn[4], const int valid[4]) {
    const size_t pe = plane_elems(c);
    const float* mu_p = prev + (size_t)pm * pe;
    const float* var_p = prev + (size_t)(pm + 1) * pe;
    const float* age_p = prev + (size_t)(pm + 2) * pe;
    float mu_k[4], var_k[4], age_k[4];
    for (int k = 0; k < 4; ++k) {
        if (!valid[k]) { mu_k[k] = var_k[k] = age_k[k] = 0.0f; continue; }
        size_t idx = (size_t)ky[k] * (size_t)c->Wb + (size_t)kx[k];
        mu_k[k] = mu_p[idx];
        var_k[k] = var_p[idx];
        age_k[k] = age_p[idx];
    }
    sgm m;
    float acc = 0.0f;
    for (int k = 0; k < 4; ++k)
        if (valid[k]) acc = fmaf(wn[k], mu_k[k], acc);
    m.mu = acc;
    acc = 0.0f;
    for (int k = 0; k < 4; ++k) {
        if (!valid[k]) continue;
        float d = m.mu - mu_k[k];
        float second = fmaf(d, d, var_k[k]);   /* var_k + (mu~ - mu_k)^2 */
        acc = fmaf(wn[k], second, acc);
    }
    m.var = acc;
    acc = 0.0f;
    for (int k = 0; k < 4; ++k)
        if (valid[k]) acc = fmaf(wn[k], age_k[k], acc);
    m.age = acc < c->p.age_cap ? acc : c->p.age_cap;
    /* S3 */
    if (c->p.decay_lambda > 0.0f && m.var > c->p.decay_var_thresh) {
        float excess = m.var - c->p.decay_var_thresh;
        m.age = m.age * decay_factor(c->p.decay_lambda, excess);
    }
    return m;
}

/* Eq. 6: V = max_{j in G_i} (mu^(t) - I_j)^2 with the UPDATED mean (App. E). */
static float block_V(float mu, const uint8_t* frame, size_t pitch, int x0, int y0, int N) {
    float V = 0.0f;
    int first = 1;
    for (int y = 0; y < N; ++y)
        for (int x = 0; x < N; ++x) {
            float e = mu - (float)frame[(size_t)(y0 + y) * pitch + (size_t)(x0 + x)];
            float e2 = e * e;
            if (first || e2 > V) V = e2;
            first = 0;
        }
    return V;
}

/* Eqs. 3, 5, 6, 7 for a matched model (R10: incremental form of Eq. 3/5 with
 * the learning rate 1/(alpha~+1) computed once, mu = fma(M - mu~, rate, mu~);
 * R22: alpha = min(alpha~+1, cap)), or the
 * App. E code rule when update_rule == 1 (R27). */
static sgm update_model(const dmsgm_oracle_ctx* c, sgm t, float M, const uint8_t* frame,
                        size_t pitch, int x0, int y0) {
    sgm r;
    if (c->p.update_rule == 0) {
        float den = t.age + 1.0f;
        float rate = 1.0f / den;                                         /* 1/(alpha~+1) */
        r.mu = fmaf(M - t.mu, rate, t.mu);                               /* Eq. 3 */
        float V = block_V(r.mu, frame, pitch, x0, y0, c->N);             /* Eq. 6 */
        r.var = fmaf(V - t.var, rate, t.var);                            /* Eq. 5 */
        r.age = den < c->p.age_cap ? den : c->p.age_cap;                 /* Eq. 7 + cap */
    } else {
        float age = t.age > 1.0f ? t.age : 1.0f;
        float alpha = 1.0f / age;                                        /* App. E */
        float keep = 1.0f - alpha;
        r.mu = keep * t.mu + alpha * M;
        float V = block_V(r.mu, frame, pitch, x0, y0, c->N);
        r.var = keep * t.var + alpha * V;
        float den = t.age + 1.0f;                                        /* P:616-618 with R22: */
        r.age = den < c->p.age_cap ? den : c->p.age_cap;                 /* min(age~+1, cap) */
    }
    return r;
}

static int step_stream(dmsgm_oracle_ctx* c, int s, const uint8_t* frame, size_t fpitch,
                       const double* h, uint8_t* mask, size_t mpitch) {
    if (c->p.form == DMSGM_ORACLE_FORM_PLAIN) return dmsgm_plain_step_stream(c, s, frame, fpitch, h, mask, mpitch);
    const int N = c->N, Wb = c->Wb, Hb = c->Hb;
    const size_t pe = plane_elems(c);
    const float* prev = stream_state(c, c->cur, s);
    float* next = stream_state(c, c->cur ^ 1, s);
    const int initialised = c->initialised[s];
    const sgm fresh_tmpl = {0.0f, c->p.var_init, 1.0f};

    for (int bj = 0; bj < Hb; ++bj) {
        for (int bi = 0; bi < Wb; ++bi) {
            const int x0 = bi * N, y0 = bj * N;
            /* S4, Eq. 4: M = (1/|G_i|) sum_{j in G_i} I_j  (integer sum, one division) */
            long sum = 0;
            for (int y = 0; y < N; ++y)
                for (int x = 0; x < N; ++x) sum += frame[(size_t)(y0 + y) * fpitch + (size_t)(x0 + x)];
            const float M = (float)sum / (float)(N * N);

            sgm A, C;
            int exposed = !initialised; /* R8: first frame of a stream */
            sgm At = fresh_tmpl, Ct = fresh_tmpl;
            if (!exposed) {
                int kx[4], ky[4], valid[4], clipped;
                float Wt[4], sumW;
                exposed = project_block(Wb, Hb, N, h, bi, bj, kx, ky, Wt, &sumW, &clipped);   /* S1 */
                if (!exposed) {
                    float wn[4];
                    for (int k = 0; k < 4; ++k) {
                        valid[k] = Wt[k] != 0.0f;
                        wn[k] = clipped ? Wt[k] / sumW : Wt[k];                            /* R6 */
                    }
                    At = mix_model(c, prev, P_MU_A, kx, ky, wn, valid);           /* S2+S3 */
                    Ct = mix_model(c, prev, P_MU_C, kx, ky, wn, valid);
                }
            }
            if (c->dump) oracle_dump_tilde(c, s, bj, bi, At, Ct, M, !exposed);   /* test probe only */
            if (exposed) {
                /* S0 / R8: A = C = (M, var_init, 1); no update this frame */
                A.mu = M; A.var = c->p.var_init; A.age = 1.0f;
                C = A;
            } else {
                /* S5, Eqs. 8-9 (App. E): tilde state, strict <, floor */
                float dA = M - At.mu;
                float gA = At.var > c->p.var_floor_match ? At.var : c->p.var_floor_match;
                int matchA = dA * dA < c->p.theta_s * gA;
                int matchC = 0;
                if (!matchA) {
                    float dC = M - Ct.mu;
                    float gC = Ct.var > c->p.var_floor_match ? Ct.var : c->p.var_floor_match;
                    matchC = dC * dC < c->p.theta_s * gC;
                }
                /* S6: update the matched model; the other keeps its tilde values (R11) */
                if (matchA) {
                    A = update_model(c, At, M, frame, fpitch, x0, y0);
                    C = Ct;
                } else if (matchC) {
                    A = At;
                    C = update_model(c, Ct, M, frame, fpitch, x0, y0);
                } else {
                    A = At;                                         /* candidate reset */
                    C.mu = M; C.var = c->p.var_init; C.age = 1.0f;
                }
                /* S7, Eq. 10: alpha_A < alpha_C  =>  A <- C, reset C */
                if (C.age > A.age) {
                    A = C;
                    C.mu = M; C.var = c->p.var_init; C.age = 1.0f;
                }
            }

            /* S8, App. E: background iff (mu_A - I)^2 <= theta_d * max(f_c, var_A) */
            for (int y = 0; y < N; ++y) {
                for (int x = 0; x < N; ++x) {
                    float I = (float)frame[(size_t)(y0 + y) * fpitch + (size_t)(x0 + x)];
                    float T;
                    if (c->p.classify_rule == 0)
                        T = c->p.theta_d * (A.var > c->p.var_floor_classify ? A.var : c->p.var_floor_classify);
                    else
                        T = c->p.theta_d * (I > c->p.var_floor_classify ? I : c->p.var_floor_classify);
                    float d = I - A.mu;
                    mask[(size_t)(y0 + y) * mpitch + (size_t)(x0 + x)] = (d * d > T) ? 255 : 0;
                }
            }

            /* S9: store into the next buffer */
            size_t idx = (size_t)bj * (size_t)Wb + (size_t)bi;
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

static int params_ok(const dmsgm_oracle_params* p) {
    if (!p) return 0;
    if (!(p->theta_s > 0.0f) || !(p->theta_d > 0.0f) || !(p->age_cap >= 1.0f)) return 0;
    if (!(p->var_init >= 0.0f) || !(p->var_floor_match > 0.0f) || !(p->var_floor_classify > 0.0f)) return 0;
    if (!(p->decay_lambda >= 0.0f) || !(p->decay_var_thresh >= 0.0f)) return 0;
    if (p->num_streams < 1) return 0;
    if (p->update_rule < 0 || p->update_rule > 1 || p->classify_rule < 0 || p->classify_rule > 1) return 0;
    if (p->form != DMSGM_ORACLE_FORM_KERNEL_ORDER && p->form != DMSGM_ORACLE_FORM_PLAIN) return 0;
    return 1;
}

int dmsgm_oracle_create(int width, int height, int block, const dmsgm_oracle_params* p,
                        dmsgm_oracle_ctx** out) {
    if (!out) return -1;
    *out = NULL;
    if (!params_ok(p)) return -1;
    if (block != 1 && block != 2 && block != 4 && block != 8 && block != 16) return -1;
    if (width <= 0 || height <= 0 || width % block || height % block) return -1; /* R1 */
    dmsgm_oracle_ctx* c = (dmsgm_oracle_ctx*)calloc(1, sizeof(*c));
    if (!c) return -2;
    c->W = width; c->H = height; c->N = block;
    c->Wb = width / block; c->Hb = height / block;
    c->S = p->num_streams;
    c->p = *p;
    size_t n = (size_t)c->S * P_NUM * plane_elems(c);
    c->state[0] = (float*)calloc(n, sizeof(float));
    c->state[1] = (float*)calloc(n, sizeof(float));
    c->initialised = (unsigned char*)calloc((size_t)c->S, 1);
    if (!c->state[0] || !c->state[1] || !c->initialised) {
        dmsgm_oracle_destroy(c);
        return -2;
    }
    *out = c;
    return 0;
}

void dmsgm_oracle_destroy(dmsgm_oracle_ctx* c) {
    if (!c) return;
    free(c->state[0]);
    free(c->state[1]);
    free(c->initialised);
    free(c);
}

int dmsgm_oracle_step_stream(dmsgm_oracle_ctx* c, int s, const uint8_t* frame, size_t fpitch,
                             const double* h, uint8_t* mask, size_t mpitch) {
    if (!c || !frame || !mask || s < 0 || s >= c->S) return -1;
    if (fpitch < (size_t)c->W || mpitch < (size_t)c->W) return -1;
    if (c->initialised[s] && !h) return -1;
    return step_stream(c, s, frame, fpitch, h, mask, mpitch);
}

int dmsgm_oracle_commit(dmsgm_oracle_ctx* c) {
    if (!c) return -1;
    memset(c->initialised, 1, (size_t)c->S);
    c->cur ^= 1;
    return 0;
}

int dmsgm_oracle_step(dmsgm_oracle_ctx* c, const uint8_t* frames, size_t fpitch,
                      const double* H, uint8_t* masks, size_t mpitch) {
    if (!c || !frames || !masks || !H) return -1;
    if (fpitch < (size_t)c->W || mpitch < (size_t)c->W) return -1;
    for (int s = 0; s < c->S; ++s) {
        int r = step_stream(c, s, frames + (size_t)s * (size_t)c->H * fpitch, fpitch, H + 9 * (size_t)s,
                            masks + (size_t)s * (size_t)c->H * mpitch, mpitch);
        if (r) return r;
    }
    return dmsgm_oracle_commit(c);
}

int dmsgm_oracle_reset(dmsgm_oracle_ctx* c, int stream) {
    if (!c || stream < -1 || stream >= c->S) return -1;
    if (stream == -1) memset(c->initialised, 0, (size_t)c->S);
    else c->initialised[stream] = 0;
    return 0;
}

int dmsgm_oracle_get_state(const dmsgm_oracle_ctx* c, int stream, float* out) {
    if (!c || !out || stream < 0 || stream >= c->S) return -1;
    memcpy(out, stream_state(c, c->cur, stream), P_NUM * plane_elems(c) * sizeof(float));
    return 0;
}

int dmsgm_oracle_set_state(dmsgm_oracle_ctx* c, int stream, const float* in) {
    if (!c || !in || stream < 0 || stream >= c->S) return -1;
    memcpy(stream_state(c, c->cur, stream), in, P_NUM * plane_elems(c) * sizeof(float));
    c->initialised[stream] = 1;
    return 0;
}

int dmsgm_oracle_is_initialised(const dmsgm_oracle_ctx* c, int stream) {
    if (!c || stream < 0 || stream >= c->S) return -1;
    return c->initialised[stream];
}

int dmsgm_oracle_mix_weights(int width, int height, int block, const double* h, int bi, int bj,
                             int* src_x, int* src_y, float* weight, float* sum_w) {
    if (!h || !src_x || !src_y || !weight || !sum_w) return -1;
    if (block < 1 || width % block || height % block) return -1;
    int clipped = 0;
    int r = project_block(width / block, height / block, block, h, bi, bj, src_x, src_y, weight, sum_w,
                          &clipped);
    return r ? 1 : (clipped ? 2 : 0);
}

int dmsgm_oracle_set_tilde_probe(dmsgm_oracle_ctx* c, float* buf) {
    if (!c) return -1;
    c->dump = buf;
    return 0;
}

float dmsgm_oracle_decay_factor(float lambda, float d) { return decay_factor(lambda, d); }

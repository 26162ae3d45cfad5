/*
 * oracle_ctx.h -- TEST INFRASTRUCTURE ONLY (see dmsgm_oracle.h).
 *
 * The oracle context shared by its two arithmetic forms:
 *   dmsgm_oracle.c  form 0, "kernel order": the canonical fp32 evaluation order of
 *                   DESIGN.md §2 (readings R5/R6/R10/R17/R18), which the CUDA path
 *                   reproduces bitwise;
 *   dmsgm_plain.c   form 1, "plain": SURVEY.md §8(c)'s literal definition (fp64
 *                   projection, every mixed sum divided by sum W, IEEE division in
 *                   Eqs. 3/5, libm exp in fp64), against which form 0 is pinned.
 * Nothing here is shared with the CUDA product path.
 */
#ifndef DMSGM_ORACLE_CTX_H
#define DMSGM_ORACLE_CTX_H

#include "dmsgm_oracle.h"

struct dmsgm_oracle_ctx {
    int W, H, N, Wb, Hb, S;
    dmsgm_oracle_params p;
    float* state[2];            /* [S][6][Hb][Wb] */
    int cur;                    /* state[cur] holds the models after frame t-1 */
    unsigned char* initialised; /* [S] */
    float* dump;                /* test probe (dmsgm_oracle_set_tilde_probe): [S][8][Hb][Wb] or NULL */
};

/* One single Gaussian model: mean mu, variance sigma, age alpha (§2.2). */
typedef struct {
    float mu;
    float var;
    float age;
} sgm;

enum { P_MU_A = 0, P_VAR_A, P_AGE_A, P_MU_C, P_VAR_C, P_AGE_C, P_NUM };

static inline size_t oracle_plane_elems(const dmsgm_oracle_ctx* c) { return (size_t)c->Wb * (size_t)c->Hb; }

static inline float* oracle_stream_state(const dmsgm_oracle_ctx* c, int buf, int s) {
    return c->state[buf] + (size_t)s * P_NUM * oracle_plane_elems(c);
}

/* Test probe: the block's tilde models (after S1-S3), M and whether it was live (not exposed). */
static inline void oracle_dump_tilde(const dmsgm_oracle_ctx* c, int s, int bj, int bi, sgm At, sgm Ct, float M,
                                     int live) {
    const size_t pe = oracle_plane_elems(c), idx = (size_t)bj * (size_t)c->Wb + (size_t)bi;
    float* d = c->dump + (size_t)s * 8 * pe;
    const float v[8] = {At.mu, At.var, At.age, Ct.mu, Ct.var, Ct.age, M, (float)live};
    for (int k = 0; k < 8; ++k) d[(size_t)k * pe + idx] = v[k];
}

/* form 1 (dmsgm_plain.c): one stream, one frame, into state[cur ^ 1] */
int dmsgm_plain_step_stream(dmsgm_oracle_ctx* c, int s, const uint8_t* frame, size_t fpitch, const double* h,
                            uint8_t* mask, size_t mpitch);

#endif
